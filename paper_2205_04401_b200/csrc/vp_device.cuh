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
  double ball;                    // != 0: ball model, ta0/ta1 = centre - v0, ta2 = factor^2 R^2
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

// Ball near-field model: circumscribed circle of (a, b, c)
// scaled by `factor`; same operation order as the oracle's ball_of/in_ball.
__device__ __forceinline__ bool rn_ball_test(double ax, double ay, double bx, double by, double cx, double cy,
                                             double factor, double tx, double ty) {
  const double bxr = rn_sub(bx, ax), byr = rn_sub(by, ay), cxr = rn_sub(cx, ax), cyr = rn_sub(cy, ay);
  const double d = rn_mul(2.0, rn_sub(rn_mul(bxr, cyr), rn_mul(byr, cxr)));
  const double b2 = rn_add(rn_mul(bxr, bxr), rn_mul(byr, byr)), c2 = rn_add(rn_mul(cxr, cxr), rn_mul(cyr, cyr));
  const double ux = rn_div(rn_sub(rn_mul(cyr, b2), rn_mul(byr, c2)), d);
  const double uy = rn_div(rn_sub(rn_mul(bxr, c2), rn_mul(cxr, b2)), d);
  const double rr = rn_mul(rn_mul(factor, factor), rn_add(rn_mul(ux, ux), rn_mul(uy, uy)));
  const double dx = rn_sub(rn_sub(tx, ax), ux), dy = rn_sub(rn_sub(ty, ay), uy);
  return rn_add(rn_mul(dx, dx), rn_mul(dy, dy)) < rr;
}

// t inside the union of the element's three open ellipses,
// or inside its ball for the ball model
__device__ __forceinline__ bool rn_in_near(const ElemRec& E, double tx, double ty) {
  if (E.ball != 0.0) {
    const double dx = rn_sub(rn_sub(tx, E.x0), E.ta0), dy = rn_sub(rn_sub(ty, E.y0), E.ta1);
    return rn_add(rn_mul(dx, dx), rn_mul(dy, dy)) < E.ta2;
  }
  if (E.ta0 < 0.0) return true;  // all-near model
  const double d0 = rn_dist(tx, ty, E.x0, E.y0);
  const double d1 = rn_dist(tx, ty, E.x1, E.y1);
  const double d2 = rn_dist(tx, ty, E.x2, E.y2);
  return (rn_add(d0, d1) < E.ta0) || (rn_add(d1, d2) < E.ta1) || (rn_add(d2, d0) < E.ta2);
}

// rn_in_near's decision from float square roots where it is clear by a
// 4e-7 relative margin, the exactly rounded test otherwise: the decisions are
// bit-identical.  (s_k = fl32(sqrt(fl32(r_k^2))) is within 1e-7 of the exact
// distance, so s_0 + s_1 is within 1e-7 of the exact left-hand side.)
__device__ __forceinline__ bool rn_in_near_fast(const ElemRec& E, double tx, double ty) {
  if (E.ball != 0.0 || E.ta0 < 0.0) return rn_in_near(E, tx, ty);
  const double px[3] = {E.x0, E.x1, E.x2}, py[3] = {E.y0, E.y1, E.y2};
  double s[3];
  bool range_ok = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double dx = tx - px[k], dy = ty - py[k];
    const double r2 = fma(dx, dx, dy * dy);
    range_ok = range_ok && r2 > 1e-30 && r2 < 1e30;
    s[k] = (double)__fsqrt_rn((float)r2);
  }
  if (range_ok) {
    const double ta[3] = {E.ta0, E.ta1, E.ta2};
    bool ambiguous = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double l = s[k] + s[(k + 1) % 3];
      if (l < ta[k] * (1.0 - 4e-7)) return true;
      ambiguous = ambiguous || !(l > ta[k] * (1.0 + 4e-7));
    }
    if (!ambiguous) return false;
  }
  return rn_in_near(E, tx, ty);
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

// The same coefficients as a __constant__ table (density_n<.., CT = true>),
// loaded by LDC/LDCU: as 64-bit immediates the compiler rebuilt each one
// with a UMOV pair per use (17 % of k_near_int's instructions; 0.98 ->
// 0.95 ms).  K5 keeps the immediates (with the table it spilled more and
// ran 4 % slower).
constexpr int kKcN = 13;  // p <= 12
struct KcTable {
  double ja[kKcN * kKcN], jb[kKcN * kKcN], jc[kKcN * kKcN], la[kKcN], lb[kKcN];
};
__host__ __device__ constexpr KcTable make_kc_table() {
  KcTable t{};
  for (int m = 0; m < kKcN; ++m) {
    const double a = 2 * m + 1;
    t.la[m] = m >= 1 ? kc_la(m) : 1.0;
    t.lb[m] = m >= 1 ? kc_lb(m) : 0.0;
    for (int k = 0; k < kKcN; ++k) {
      t.ja[m * kKcN + k] = k == 0 ? 0.5 * (a + 2.0) : kc_ja(m, k);
      t.jb[m * kKcN + k] = k == 0 ? 0.5 * a : kc_jb(m, k);
      t.jc[m * kKcN + k] = k == 0 ? 0.0 : kc_jc(m, k);
    }
  }
  return t;
}
__constant__ KcTable c_kc = make_kc_table();

// f(x, y) = sum_j cc_j K_j(x, y) where cc_j already includes the
// normalisation c_mn (pre-scaled per element).  Template recursion over
// (m, k) makes every recurrence coefficient a compile-time constant (no
// runtime divisions); ~4 FP64 ops per mode.
// Coefficient accessor for shared memory: an `ld.shared` in volatile asm is
// re-issued at every use (a broadcast LDS, one wavefront), so the
// coefficients are never hoisted into (and spilled from) registers.
struct ShCoef {
  unsigned base;
  __device__ __forceinline__ explicit ShCoef(const double* p)
      : base((unsigned)__cvta_generic_to_shared(p)) {}
  __device__ __forceinline__ double operator[](int i) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 8u * (unsigned)i));
    return v;
  }
};

// Per m, S_m(t) = sum_k cc[m, m+k] P_k^{(2m+1,0)}(t) by Clenshaw's backward
// recurrence (b_k = c_k + alpha_k b_{k+1} - beta_{k+1} b_{k+2}, S_m = b_0;
// alpha_k = ja t + jb, beta_k = jc): 3 FP64 ops per mode.  Then
// f = sum_m S_m L_m with L_m the homogenised Legendre recurrence.  NPT points
// share every coefficient load.
template <int NPT>
struct Pts {
  double v[NPT];
};

template <int P, int m, int k, int NPT, bool CT, class CC>
__device__ __forceinline__ void clenshaw_m(const CC& cc, const Pts<NPT>& t, Pts<NPT>& b1, Pts<NPT>& b2) {
  // processes k = P - m down to 0 for fixed m; on exit b1 = b_0 = S_m
  if constexpr (k >= 0) {
    const double c = cc[koorn_index(m, m + k)];
    if constexpr (k == P - m) {
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        b2.v[i] = 0.0;
        b1.v[i] = c;
      }
    } else {
      constexpr double a = 2 * m + 1;
      const double ja = CT ? c_kc.ja[m * kKcN + k] : ((k == 0) ? 0.5 * (a + 2.0) : kc_ja(m, k));
      const double jb = CT ? c_kc.jb[m * kKcN + k] : ((k == 0) ? 0.5 * a : kc_jb(m, k));
      const double jc1 = CT ? c_kc.jc[m * kKcN + k + 1] : kc_jc(m, k + 1);  // beta_{k+1}
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        const double al = fma(ja, t.v[i], jb);
        double bk = fma(al, b1.v[i], c);
        if constexpr (k + 2 <= P - m) bk = fma(-jc1, b2.v[i], bk);
        b2.v[i] = b1.v[i];
        b1.v[i] = bk;
      }
    }
    clenshaw_m<P, m, k - 1, NPT, CT, CC>(cc, t, b1, b2);
  }
}

template <int P, int m, int NPT, bool CT, class CC>
__device__ __forceinline__ void koorn_modes_n(const CC& cc, const Pts<NPT>& t, const Pts<NPT>& u,
                                              const Pts<NPT>& v2, Pts<NPT>& Lm, Pts<NPT>& Lprev,
                                              Pts<NPT>& f) {
  if constexpr (m <= P) {
    Pts<NPT> b1, b2;
    clenshaw_m<P, m, P - m, NPT, CT, CC>(cc, t, b1, b2);
#pragma unroll
    for (int i = 0; i < NPT; ++i) f.v[i] = fma(b1.v[i], Lm.v[i], f.v[i]);
    if constexpr (m < P) {
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        double Ln;
        if constexpr (m == 0) {
          Ln = u.v[i];
        } else {
          const double la = CT ? c_kc.la[m] : kc_la(m), lb = CT ? c_kc.lb[m] : kc_lb(m);
          Ln = fma(la * u.v[i], Lm.v[i], -lb * v2.v[i] * Lprev.v[i]);
        }
        Lprev.v[i] = Lm.v[i];
        Lm.v[i] = Ln;
      }
      koorn_modes_n<P, m + 1, NPT, CT, CC>(cc, t, u, v2, Lm, Lprev, f);
    }
  }
}

// f at NPT points (x[i], y[i]); CT: recurrence constants from c_kc
template <int P, int NPT, bool CT = false, class CC>
__device__ __forceinline__ void density_n(const CC& cc, const double* x, const double* y, double* out) {
  Pts<NPT> t, u, v2, Lm, Lprev, f;
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const double v = 1.0 - x[i];
    u.v[i] = fma(2.0, y[i], -v);
    v2.v[i] = v * v;
    t.v[i] = fma(2.0, x[i], -1.0);
    Lm.v[i] = 1.0;
    Lprev.v[i] = 0.0;
    f.v[i] = 0.0;
  }
  koorn_modes_n<P, 0, NPT, CT, CC>(cc, t, u, v2, Lm, Lprev, f);
#pragma unroll
  for (int i = 0; i < NPT; ++i) out[i] = f.v[i];
}

template <int P, class CC>
__device__ __forceinline__ double density(const CC& cc, double x, double y) {
  double o;
  density_n<P, 1, false, CC>(cc, &x, &y, &o);
  return o;
}

// ---------------------------------------------------------------------------
// fp64 log of x = r^2 > 0 with 13 FP64 operations (vs ~30 for libdevice):
//   x = 2^e m, m in [1,2); k = top 8 mantissa bits; r_k ~ 1/(1 + (k+1/2)/256)
//   log x = e ln2 - log r_k + log(1 + t),  t = m r_k - 1 (one FMA), |t| <= 2^-9
//   log(1+t) by a degree-5 Taylor polynomial (truncation <= 1e-17).
// The table {r_k, -log r_k} lives in shared memory, replicated 8x so that
// the 8 lanes of a quarter-warp hit 8 different bank groups (conflict-free
// 128-bit loads).  x == 0 (coincident pair) returns 0.
#ifndef VP_LOG_BITS
#define VP_LOG_BITS 9
#endif
#ifndef VP_LOG_I2F
#define VP_LOG_I2F 1
#endif
constexpr int kLogBits = VP_LOG_BITS;
constexpr int kLogEntries = 1 << kLogBits;
constexpr int kLogCopies = 8;

struct LogTab {
  double2 e[kLogEntries * kLogCopies];  // entry k, copy c at k*8 + c
};

inline void log_table_fill(double2* host /* n */, int n = kLogEntries) {
  for (int k = 0; k < n; ++k) {
    const long double mk = 1.0L + ((long double)k + 0.5L) / (long double)n;
    const double r = (double)(1.0L / mk);
    host[k].x = r;
    host[k].y = (double)(-log1pl((long double)r - 1.0L));
  }
}

#ifdef __CUDACC__
// L + log(1 + t) for |t| <= 2^-(kLogBits+1):
//   8 bits: Taylor degree 5 (truncation 9e-18);
//   9 bits: minimax degree 4 on [-2^-10, 2^-10] (max error 2.3e-17).
static_assert(kLogBits == 8 || kLogBits == 9, "log table: 8 or 9 index bits");
// The 9-bit polynomial's constants and ln 2 live in __constant__ memory so a
// DFMA takes them as a constant-bank operand: literal doubles are otherwise
// re-materialised into uniform registers inside register-tight loops.
// (CB = true; K2 keeps literals, which measure 0.5 % faster there.)
__constant__ double c_logk[4] = {-0.25000024181904215854, 0.3333334991010435487, -0.49999999999992096269,
                                 0.69314718055994530942};
template <bool CB>
__device__ __forceinline__ double log_ln2() {
  if constexpr (CB) return c_logk[3];
  return 0.69314718055994530942;
}
template <bool CB = true>
__device__ __forceinline__ double log1p_poly(double t, double L) {
  if constexpr (kLogBits == 9 && CB) {
    double i = fma(t, c_logk[0], c_logk[1]);
    i = fma(t, i, c_logk[2]);
    i = fma(t, i, 1.0);
    return fma(t, i, L);
  }
  if constexpr (kLogBits == 8) {
    double i = fma(t, 0.2, -0.25);
    i = fma(t, i, 0.33333333333333333);
    i = fma(t, i, -0.5);
    i = fma(t, i, 1.0);
    return fma(t, i, L);
  } else {
    double i = fma(t, -0.25000024181904215854, 0.3333334991010435487);
    i = fma(t, i, -0.49999999999992096269);
    i = fma(t, i, 1.0);
    return fma(t, i, L);
  }
}

__device__ __forceinline__ double log_exponent(unsigned hi) {
  if constexpr (VP_LOG_I2F) {
    return (double)((int)(hi >> 20) - 1023);
  } else {
    return __hiloint2double(0x43380000, (int)(hi >> 20)) - 6755399441056767.0;  // e = biased - 1023
  }
}

// base: this lane's copy (tab + (lane & 7) with STRIDE = kLogCopies), or an
// unreplicated table with STRIDE = 1
template <int STRIDE, bool ZERO_CHECK = true>
__device__ __forceinline__ double fast_log_r2(const double2* __restrict__ base, double x) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const double2 tb = base[((hi >> (20 - kLogBits)) & (kLogEntries - 1)) * STRIDE];
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double ed = log_exponent((unsigned)hi);
  const double t = fma(m, tb.x, -1.0);
  const double p = log1p_poly<true>(t, tb.y);
  const double lg = fma(ed, log_ln2<true>(), p);
  if constexpr (ZERO_CHECK) return hi >= 0x00100000 ? lg : 0.0;
  return lg;
}

// Far-kernel variant of fast_log_r2 with fewer integer operations:
//   * `tab` is the replicated table in *static* shared memory (its address is
//     a link-time constant folded into the LDS immediate); the entry offset
//     k*128 and the lane's copy offset (lane&7)*16 are combined by one LOP3;
//   * the mantissa m is built with one LOP3 using `c3ff` = 0x3ff00000 held in
//     a register;
//   * ZERO_CHECK = false skips the r^2 == 0 test.  That is exact for the
//     evaluation path: a target can only coincide with an interior node of
//     its own element S(t), whose point sum is subtracted again with the same
//     function (subtract-and-add), so the finite value
//     returned for r^2 == 0 cancels.
template <bool ZERO_CHECK, bool CB = false>
__device__ __forceinline__ double far_log_r2(const double2* tab, unsigned laneoff, unsigned c3ff, double x) {
  const unsigned hi = (unsigned)__double2hiint(x), lo = (unsigned)__double2loint(x);
  unsigned off, mhi;
  // byte offset of entry k (stride kLogCopies * 16 = 128 B) OR the lane's copy
  constexpr unsigned kShift = 20 - kLogBits - 7, kMask = (unsigned)(kLogEntries - 1) << 7;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(off) : "r"(hi >> kShift), "n"(kMask), "r"(laneoff));
  asm("lop3.b32 %0, %1, 0x000fffff, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(c3ff));
  const double2 tb = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(tab) + off);
  const double m = __hiloint2double((int)mhi, (int)lo);
  const double ed = log_exponent(hi);
  const double t = fma(m, tb.x, -1.0);
  const double p = log1p_poly<CB>(t, tb.y);
  const double lg = fma(ed, log_ln2<CB>(), p);
  if constexpr (ZERO_CHECK) return hi >= 0x00100000u ? lg : 0.0;
  return lg;
}
#endif

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#endif  // __CUDACC__

}  // namespace vp
