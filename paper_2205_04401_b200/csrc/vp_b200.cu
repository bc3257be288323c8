// vp_b200.cu -- B200 (sm_100a) evaluator for the 2-D log-kernel volume
// potential: kernels K1-K5 and the C-ABI of include/vp.h.
//
//   K1 k_sources   ChargeSystem strengths       FP64, tiny
//   K2 k_far       direct far sum          FP64 pipe
//   K3 k_lists     S(t), N(t) CSR      HBM/latency
//   K4 k_near      near_eval - point sum         FP64 pipe
//   K5 k_self      self_eval - point sum         FP64 pipe
//   k_assemble     subtract-and-add
//
// Data stays resident in HBM inside the context; every per-target result is
// produced by a fixed-order reduction, so u is deterministic run to run and
// independent of how targets are sharded across GPUs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cub/cub.cuh>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "vp.h"
#include "vp_setup.h"
#include "vp_device.cuh"
#include "vp_curve.cuh"

using namespace vp;

namespace {

constexpr int kMaxPdev = 12;
constexpr int kMaxModes = (kMaxPdev + 1) * (kMaxPdev + 2) / 2;  // 91
// K5 samples the density from monomial coefficients about the reference
// centroid for p <= kMonoMaxP (27 DFMA per point at p = 6 instead of the
// ~120-op Koornwinder recurrence); the monomial basis costs a factor
// (|K| coefficient growth) 1e2 / 1e3 in rounding at p = 6 / 8 for rough
// densities, none for smooth ones; above p = 8 the growth is
// 1e5+, so K5 keeps the recurrence.
constexpr int kMonoMaxP = 8;
constexpr int kMonoMaxModes = (kMonoMaxP + 1) * (kMonoMaxP + 2) / 2;  // 45
constexpr double kMonoC0 = 1.0 / 3.0;  // expansion centre (c0, c0), exactly this double
constexpr int kMaxFar = 1024;
constexpr int kMaxNearRule = 256;
constexpr int kMaxGL = 64;
constexpr int kMaxGGQ = 32;

__constant__ double c_cn[kMaxModes];  // Koornwinder normalisation c_mn by index

struct RulesDev {
  int len_q, len_n, n_l, n_g1, n_n, q;
  int near_model, pad_;   // 0 precise, 1 ball
  double ball_factor;
  double far_x[kMaxFar], far_y[kMaxFar], far_w[kMaxFar];
  double near_x[kMaxNearRule], near_y[kMaxNearRule], near_w[kMaxNearRule];
  double gl_x[kMaxGL], gl_w[kMaxGL];
  double ggq_r[kMaxGGQ], ggq_w[kMaxGGQ], ggq_lr[kMaxGGQ];
  double kd[kMaxNearDepth + 2];  // 4^{-d/N_n}
};

struct GridDev {
  double x0, y0, cs, inv_cs;
  int nx, ny;
};

// curved elements (vp_curve.cuh): element -> curve, blending geometry
__device__ __forceinline__ int curve_id_of(const CurvesDev& CV, int64_t e) { return CV.ecurve ? CV.ecurve[e] : -1; }
__device__ __forceinline__ CurveRef curve_of(const CurvesDev& CV, int c) {
  return CurveRef{CV.cx + (int64_t)c * (CV.D + 1), CV.cy + (int64_t)c * (CV.D + 1), CV.D, CV.len[c]};
}
__device__ __forceinline__ BlendGeom bgeom_of(const ElemRec& E) {
  return BlendGeom{E.x0, E.y0, E.x1, E.y1, E.x2, E.y2};
}

// containment in a curved element (oracle ref_coords, curved branch): the
// chord's affine inverse seeds 12 Newton steps of the blending-map inverse;
// a residual above 1e-9 L never counts as inside
__device__ __forceinline__ bool rn_locate_curved(const ElemRec& E, const CurveRef& C, double tx, double ty,
                                                 double& xi, double& eta) {
  const double dx = rn_sub(tx, E.x0), dy = rn_sub(ty, E.y0);
  xi = rn_add(rn_mul(E.i00, dx), rn_mul(E.i01, dy));
  eta = rn_add(rn_mul(E.i10, dx), rn_mul(E.i11, dy));
  const BlendGeom B = bgeom_of(E);
  blend_inverse<true>(B, C, tx, ty, xi, eta);
  double x, y;
  blend<true>(B, C, xi, eta, x, y);
  const double rx = rn_sub(tx, x), ry = rn_sub(ty, y);
  const double tolr = rn_mul(1e-9, C.L);
  if (!(rn_add(rn_mul(rx, rx), rn_mul(ry, ry)) <= rn_mul(tolr, tolr))) return false;
  const double l0 = rn_sub(rn_sub(1.0, xi), eta);
  return xi >= -kBaryTol && eta >= -kBaryTol && l0 >= -kBaryTol;
}

// K1 for curved elements: overwrite the sources of the listed curved
// elements with y_i = rho(xi_i), q_i *= |J(xi_i)| / det (k_sources used the chord)
__global__ void k_sources_curved(int64_t n, const int32_t* __restrict__ celist, int len_q,
                                 const ElemRec* __restrict__ el, CurvesDev CV, const RulesDev* __restrict__ R,
                                 double* __restrict__ sx, double* __restrict__ sy, double* __restrict__ sq) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n * len_q) return;
  const int64_t k = s / len_q;
  const int i = (int)(s - k * len_q);
  const int64_t e = celist[k];
  const ElemRec& T = el[e];
  const CurveRef C = curve_of(CV, CV.ecurve[e]);
  double x, y, J[4];
  blend_jac<false>(bgeom_of(T), C, R->far_x[i], R->far_y[i], x, y, J);
  const int64_t o = e * len_q + i;
  sx[o] = x;
  sy[o] = y;
  sq[o] = sq[o] * (fabs(J[0] * J[3] - J[1] * J[2]) / T.det);
}

// ---------------------------------------------------------------------------
// K1: point sources y_i = rho_T(xi_i), q_i = w_i |J_T| f_T(xi_i) / (4 pi).
// f_T(xi_i) = V[i,:] . c_T with V the Koornwinder values at the far nodes.
__global__ void k_sources(int64_t E, int len_q, int M, const ElemRec* __restrict__ el,
                          const double* __restrict__ coeffs, const double* __restrict__ V,
                          const RulesDev* __restrict__ R, double* __restrict__ sx,
                          double* __restrict__ sy, double* __restrict__ sq) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= E * len_q) return;
  const int64_t e = s / len_q;
  const int i = (int)(s - e * len_q);
  const ElemRec& T = el[e];
  const double xi = R->far_x[i], eta = R->far_y[i];
  sx[s] = T.x0 + (xi * T.e1x + eta * T.e2x);
  sy[s] = T.y0 + (xi * T.e1y + eta * T.e2y);
  const double* c = coeffs + e * M;
  const double* v = V + (int64_t)i * M;
  double f = 0.0;
  for (int j = 0; j < M; ++j) f = fma(c[j], v[j], f);
  sq[s] = (R->far_w[i] * T.det) * f * kInv4Pi;
}

// Per-element monomial coefficients of the density about the reference
// centroid c0 = (1/3, 1/3) (double-rounded), for the self kernel's density
// samples: mono[e, i] = sum_j coeffs[e, j] Kmon[j, i], Kmon the exact
// (long double) expansion of c_j K_j (upload_self_tab).  p <= kMonoMaxP only.
__global__ void __launch_bounds__(256) k_mono(int64_t E, int M, const double* __restrict__ coeffs,
                                              const double* __restrict__ kmon, double* __restrict__ mono) {
  __shared__ double sk[kMonoMaxModes * kMonoMaxModes];
  for (int i = threadIdx.x; i < M * M; i += blockDim.x) sk[i] = kmon[i];
  __syncthreads();
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= E * M) return;
  const int64_t e = o / M;
  const int i = (int)(o - e * M);
  const double* c = coeffs + e * M;
  double s0 = 0.0, s1 = 0.0;
  int j = 0;
  for (; j + 2 <= M; j += 2) {
    s0 = fma(c[j], sk[j * M + i], s0);
    s1 = fma(c[j + 1], sk[(j + 1) * M + i], s1);
  }
  if (j < M) s0 = fma(c[j], sk[j * M + i], s0);
  mono[o] = s0 + s1;
}

// ---------------------------------------------------------------------------
// element binning for the list build: every element is entered in each grid
// cell its near-field bbox overlaps.  Cell size in units of the median
// near-field extent B: a target scans ~ (1 + cs / B)^2 bboxes' worth of
// elements, the bins hold ~ (1 + B / cs)^2 entries per element.
constexpr double kGridScale = 0.25;
__device__ __forceinline__ int cell_coord(double x, double x0, double inv_cs, int n) {
  const double f = floor(rn_mul(rn_sub(x, x0), inv_cs));
  int c = f < 0.0 ? 0 : (f >= (double)n ? n - 1 : (int)f);
  return c;
}

__global__ void k_bin_count(int64_t E, const ElemRec* __restrict__ el, GridDev g,
                            int64_t* __restrict__ cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const ElemRec& T = el[e];
  if (T.ball == 0.0 && T.ta0 < 0.0) {  // all-near: scanned by every target instead
    cnt[e] = 0;
    return;
  }
  const int cx0 = cell_coord(T.bx0, g.x0, g.inv_cs, g.nx), cx1 = cell_coord(T.bx1, g.x0, g.inv_cs, g.nx);
  const int cy0 = cell_coord(T.by0, g.y0, g.inv_cs, g.ny), cy1 = cell_coord(T.by1, g.y0, g.inv_cs, g.ny);
  cnt[e] = (int64_t)(cx1 - cx0 + 1) * (cy1 - cy0 + 1);
}

__global__ void k_bin_fill(int64_t E, const ElemRec* __restrict__ el, GridDev g,
                           const int64_t* __restrict__ off, int32_t* __restrict__ keys,
                           int32_t* __restrict__ vals) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const ElemRec& T = el[e];
  if (T.ball == 0.0 && T.ta0 < 0.0) return;
  const int cx0 = cell_coord(T.bx0, g.x0, g.inv_cs, g.nx), cx1 = cell_coord(T.bx1, g.x0, g.inv_cs, g.nx);
  const int cy0 = cell_coord(T.by0, g.y0, g.inv_cs, g.ny), cy1 = cell_coord(T.by1, g.y0, g.inv_cs, g.ny);
  int64_t o = off[e];
  for (int cy = cy0; cy <= cy1; ++cy)
    for (int cx = cx0; cx <= cx1; ++cx) {
      keys[o] = cy * g.nx + cx;
      vals[o] = (int32_t)e;
      ++o;
    }
}

__global__ void k_cell_ranges(int64_t n, const int32_t* __restrict__ keys,
                              int64_t* __restrict__ beg, int64_t* __restrict__ end) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t k = keys[i];
  if (i == 0 || keys[i - 1] != k) beg[k] = i;
  if (i == n - 1 || keys[i + 1] != k) end[k] = i + 1;
}

// ---------------------------------------------------------------------------
// K3: S(t) (lowest containing id) and N(t) (ascending) for every target.
// Candidates = the elements binned in t's cell merged with the all-near list.
// CURVED: the mesh has curved elements (their Newton locate is inlined only
// then; straight meshes run at 4 -> 8 resident blocks with 124 -> <= 64 registers)
template <bool FILL, bool CURVED>
__global__ void __launch_bounds__(128, CURVED ? 1 : 8)
    k_lists(int64_t T, const double2* __restrict__ txy,
                        const ElemRec* __restrict__ el, const float4* __restrict__ bbf, GridDev g,
                        const int64_t* __restrict__ cbeg, const int64_t* __restrict__ cend,
                        const int32_t* __restrict__ celems, const int32_t* __restrict__ allnear,
                        int n_allnear, int32_t* __restrict__ self_out,
                        int64_t* __restrict__ cnt_out, const int64_t* __restrict__ off,
                        int32_t* __restrict__ ids, double2* __restrict__ self_ref, CurvesDev CV,
                        const int32_t* __restrict__ tlist, int32_t* __restrict__ scratch, int cap,
                        int32_t* __restrict__ over, unsigned* __restrict__ n_over, int* __restrict__ nonfinite) {
  // count pass: also keeps the first `cap` ids of N(t) in scratch[t * cap ..]
  // and lists the targets with more (walked again by the fill pass over tlist);
  // flags non-finite targets (the evaluation's input check, on the device)
  const int64_t ti = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ti >= T) return;
  const int64_t t = tlist ? tlist[ti] : ti;
  const double2 p = txy[t];
  const double tx = p.x, ty = p.y;
  if (nonfinite && !(isfinite(tx) && isfinite(ty))) *nonfinite = 1;
  int64_t b = 0, e = 0;
  const double fx = floor(rn_mul(rn_sub(tx, g.x0), g.inv_cs));
  const double fy = floor(rn_mul(rn_sub(ty, g.y0), g.inv_cs));
  if (fx >= 0.0 && fy >= 0.0 && fx < (double)g.nx && fy < (double)g.ny) {
    const int c = (int)fy * g.nx + (int)fx;
    b = cbeg[c];
    e = cend[c];
  }
  int32_t self = -1;
  double sxi = 0.0, seta = 0.0;
  int64_t n = 0;
  int64_t o = FILL ? off[t] : 0;
  int ia = 0;
  while (b < e || ia < n_allnear) {
    int32_t id;
    const int32_t cb = b < e ? celems[b] : INT32_MAX;
    const int32_t ca = ia < n_allnear ? allnear[ia] : INT32_MAX;
    if (cb <= ca) {
      id = cb;
      ++b;
      if (ca == cb) ++ia;
    } else {
      id = ca;
      ++ia;
    }
    // the element's near-field bbox rounded outward to float (all-near: the
    // whole plane) rejects most candidates without touching the 192-B record
    const float4 bb = bbf[id];
    if (!(tx >= (double)bb.x && tx <= (double)bb.z && ty >= (double)bb.y && ty <= (double)bb.w)) continue;
    const ElemRec& R = el[id];
    if (self < 0) {
      double xi, eta;
      const int cid = CURVED ? curve_id_of(CV, id) : -1;
      if (cid < 0 ? rn_locate(R, tx, ty, xi, eta) : rn_locate_curved(R, curve_of(CV, cid), tx, ty, xi, eta)) {
        self = id;
        sxi = xi;
        seta = eta;
        continue;
      }
    }
    if (rn_in_near_fast(R, tx, ty)) {
      if (FILL) ids[o++] = id;
      else if (n < cap) scratch[t * cap + n] = id;
      ++n;
    }
  }
  if (!FILL) {
    cnt_out[t] = n;
    self_out[t] = self;
    if (self_ref) self_ref[t] = make_double2(sxi, seta);
    if (n > cap) over[atomicAdd(n_over, 1u)] = (int32_t)t;
  }
}

__global__ void k_lists_copy(int64_t T, const int64_t* __restrict__ off, int cap,
                             const int32_t* __restrict__ scratch, int32_t* __restrict__ ids) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int64_t o = off[t], n = off[t + 1] - o;
  if (n > cap) return;
  for (int64_t i = 0; i < n; ++i) ids[o + i] = scratch[t * cap + i];
}

__global__ void k_pair_tgt(int64_t T, const int64_t* __restrict__ off, int32_t* __restrict__ pt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  for (int64_t p = off[t]; p < off[t + 1]; ++p) pt[p] = (int32_t)t;
}

// ---------------------------------------------------------------------------
// K2: u_far[t] = sum_j q_j log r_tj^2 (coincident pairs contribute 0).
// Sources are staged through shared memory and broadcast to the block's
// targets; each thread keeps FAR_R targets in registers.  The source range
// is split over gridDim.y; partials are reduced in fixed order.
#ifndef VP_FAR_R
#define VP_FAR_R 8
#endif
#ifndef VP_NEAR_MINB
#define VP_NEAR_MINB 2
#endif
#ifndef VP_SELF_MINB
#define VP_SELF_MINB 5
#endif
#ifndef VP_FAR_MINB
#define VP_FAR_MINB 2
#endif
#ifndef VP_FAR_UNROLL
#define VP_FAR_UNROLL 2
#endif
// K2's own log table: 2^VP_FAR_LOG_BITS entries replicated VP_FAR_COPIES
// times (lane & (copies - 1) picks the copy).  With 11 index bits |t| <=
// 2^-12 and a degree-3 minimax polynomial t + c2 t^2 + c3 t^3 is exact to
// 1.9e-16 (absolute, log(1+t)), one DFMA fewer per pair than the 9-bit
// table's degree-4 polynomial shared by the other kernels.
#ifndef VP_FAR_LOG_BITS
#define VP_FAR_LOG_BITS 10
#endif
#ifndef VP_FAR_COPIES
#define VP_FAR_COPIES 8
#endif
// a table above 64 KB leaves room for one block per SM: 512 threads, so the
// SM still holds 16 warps
#if (1 << VP_FAR_LOG_BITS) * VP_FAR_COPIES * 16 > 65536
#undef VP_FAR_MINB
#define VP_FAR_MINB 1
#ifndef VP_FAR_THREADS
#define VP_FAR_THREADS 512
#endif
#endif
#ifndef VP_FAR_THREADS
#define VP_FAR_THREADS 256
#endif
constexpr int FAR_THREADS = VP_FAR_THREADS;
constexpr int FAR_R = VP_FAR_R;      // targets per thread (register tile)
constexpr int FAR_TILE = 256;        // sources per shared-memory tile
constexpr int kFarUnroll = VP_FAR_UNROLL;
constexpr int kFarLogBits = VP_FAR_LOG_BITS;
constexpr int kFarLogEntries = 1 << kFarLogBits;
constexpr int kFarCopies = VP_FAR_COPIES;
static_assert(kFarLogBits >= 9 && kFarLogBits <= 11, "far log table: 9..11 index bits");
static_assert(kFarCopies == 2 || kFarCopies == 4 || kFarCopies == 8, "far log table copies");

__device__ double2 g_logtab[kLogEntries];      // {r_k, -log r_k}, filled at vp_create
__device__ double2 g_fartab[kFarLogEntries];   // the same for K2's table

// log r^2 for K2 (see far_log_r2 in vp_device.cuh for the bit manipulation)
template <bool ZERO_CHECK>
__device__ __forceinline__ double far_log_k2(const double2* tab, unsigned laneoff, unsigned c3ff, double x) {
  if constexpr (kFarLogBits == 9 && kFarCopies == kLogCopies) {
    return far_log_r2<ZERO_CHECK>(tab, laneoff, c3ff, x);
  } else {
    const unsigned hi = (unsigned)__double2hiint(x), lo = (unsigned)__double2loint(x);
    unsigned off, mhi;
    constexpr int kStrideLog = kFarCopies == 8 ? 7 : kFarCopies == 4 ? 6 : 5;  // entry stride 16 * copies
    constexpr unsigned kShift = 20 - kFarLogBits - kStrideLog;
    constexpr unsigned kMask = (unsigned)(kFarLogEntries - 1) << kStrideLog;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(off) : "r"(hi >> kShift), "n"(kMask), "r"(laneoff));
    asm("lop3.b32 %0, %1, 0x000fffff, %2, 0xEA;" : "=r"(mhi) : "r"(hi), "r"(c3ff));
    const double2 tb = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(tab) + off);
    const double m = __hiloint2double((int)mhi, (int)lo);
    const double ed = log_exponent(hi);
    const double t = fma(m, tb.x, -1.0);
    double p;
    if constexpr (kFarLogBits == 11) {  // minimax on |t| <= 2^-12 (1.002x): 1.9e-16
      double i = fma(t, 0.33333334272003357, -0.5000000117277289);
      i = fma(t, i, 1.0);
      p = fma(t, i, tb.y);
    } else if constexpr (kFarLogBits == 10) {  // minimax on |t| <= 2^-11: 3.6e-15
      double i = fma(t, 0.33333338120707445, -0.5000000598513419);
      i = fma(t, i, 1.0);
      p = fma(t, i, tb.y);
    } else {
      p = log1p_poly<false>(t, tb.y);
    }
    const double lg = fma(ed, 0.69314718055994530942, p);
    if constexpr (ZERO_CHECK) return hi >= 0x00100000u ? lg : 0.0;
    return lg;
  }
}

template <bool ZERO_CHECK, int R = FAR_R>
__global__ void __launch_bounds__(FAR_THREADS, VP_FAR_MINB)
    k_far(int64_t T, const double2* __restrict__ txy, int64_t S, const double* __restrict__ sx,
          const double* __restrict__ sy, const double* __restrict__ sq, int64_t chunk,
          double* __restrict__ part, unsigned c3ff) {
  extern __shared__ __align__(16) unsigned char fsm[];
  double2* tab = reinterpret_cast<double2*>(fsm);  // kFarLogEntries x kFarCopies
  double2* sxy = tab + kFarLogEntries * kFarCopies;
  double* ssq = reinterpret_cast<double*>(sxy + FAR_TILE);
  for (int i = threadIdx.x; i < kFarLogEntries * kFarCopies; i += FAR_THREADS) tab[i] = g_fartab[i / kFarCopies];
  const unsigned laneoff = 16u * (threadIdx.x & (kFarCopies - 1));
  const int64_t tb = (int64_t)blockIdx.x * (FAR_THREADS * R) + threadIdx.x;
  double tx[R], ty[R], acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t t = tb + (int64_t)r * FAR_THREADS;
    const double2 p = t < T ? txy[t] : make_double2(0.0, 0.0);
    tx[r] = p.x;
    ty[r] = p.y;
    acc[r] = 0.0;
  }
  const int64_t s0 = (int64_t)blockIdx.y * chunk;
  const int64_t s1 = min(S, s0 + chunk);
  for (int64_t base = s0; base < s1; base += FAR_TILE) {
    const int n = (int)min((int64_t)FAR_TILE, s1 - base);
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += FAR_THREADS) {
      sxy[j] = make_double2(sx[base + j], sy[base + j]);
      ssq[j] = sq[base + j];
    }
    __syncthreads();
#pragma unroll (kFarUnroll)
    for (int j = 0; j < n; ++j) {
      const double2 ps = sxy[j];
      const double q = ssq[j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double dx = tx[r] - ps.x, dy = ty[r] - ps.y;
        const double r2 = fma(dx, dx, dy * dy);
        acc[r] = fma(q, far_log_k2<ZERO_CHECK>(tab, laneoff, c3ff, r2), acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t t = tb + (int64_t)r * FAR_THREADS;
    if (t < T) part[(int64_t)blockIdx.y * T + t] = acc[r];
  }
}


#include "vp_fmm.cuh"

__global__ void k_far_reduce(int64_t T, int nsplit, const double* __restrict__ part,
                             double* __restrict__ u) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  double s = 0.0;
  for (int k = 0; k < nsplit; ++k) s += part[(int64_t)k * T + t];
  u[t] = s;
}

// sum_{i in T} q_i log r^2 of element e's sources, warp-cooperative
// exact_zero = false inside the evaluation: a coincident pair (target = node of
// its own element) contributes the same finite value here as in the far sum
// (k_far / k_fmm_eval with ZERO_CHECK=false), so it cancels, as the oracle's
// skipped pair does.  The per-pair API (vp_near_pairs / vp_self_pairs) uses
// exact_zero = true so its point sum matches SPEC.md:575 on its own.
// ltab: a single-copy table (STRIDE 1) or this lane's copy of the replicated
// one (tab + (lane & 7), STRIDE kLogCopies)
template <int STRIDE = 1>
__device__ __forceinline__ double warp_point_sum(int lane, int64_t e, int len_q, double tx,
                                                 double ty, const double* __restrict__ sx,
                                                 const double* __restrict__ sy,
                                                 const double* __restrict__ sq,
                                                 const double2* __restrict__ ltab, bool exact_zero) {
  double s = 0.0;
  for (int i = lane; i < len_q; i += 32) {
    const int64_t k = e * len_q + i;
    const double dx = tx - sx[k], dy = ty - sy[k];
    const double r2 = fma(dx, dx, dy * dy);
    const double lg = exact_zero ? fast_log_r2<STRIDE, true>(ltab, r2) : fast_log_r2<STRIDE, false>(ltab, r2);
    s = fma(sq[k], lg, s);
  }
  return warp_sum(s);
}

// ---------------------------------------------------------------------------
// K4: near_eval in two stages.
//  K4a k_near_leaves<FILL>: one thread per (target, element) pair runs the
//      4-way midpoint subdivision depth-first and counts / writes its accepted
//      leaves as path codes (2 bits per level, depth in the top 6 bits).  The
//      leaf SET and every counter are the oracle's; the ORDER differs (the
//      four children of a node are tested together and the accepted ones
//      emitted at once), which only reorders the per-pair sums.
//  K4b k_near_int<P>: one warp per pair integrates the pair's leaves with the
//      N_n rule, lanes over (leaf, node) two nodes at a time, and subtracts
//      the element's far-field point sum.
constexpr int kMaxPathDepth = 29;
constexpr int NEAR_WARPS = 8;
constexpr int kStackCap = 3 * kMaxPathDepth + 4;
constexpr unsigned long long kPathMask = (1ull << 58) - 1ull;
// A CACHED leaf (depth <= D <= 6, path <= 12 bits) also carries its element
// id in bits 16..47, so the evaluation kernels read it with the code instead
// of walking the pair offsets and pair_elem.
constexpr unsigned long long kCPathMask = 0xFFFFull;
__device__ __forceinline__ unsigned long long tag_cached(unsigned long long code, int32_t e) {
  return code | ((unsigned long long)(uint32_t)e << 16);
}
__device__ __forceinline__ int32_t cached_elem(unsigned long long code) { return (int32_t)(uint32_t)(code >> 16); }

__device__ __forceinline__ void decode_path(unsigned long long path, int d, double& ax, double& ay,
                                            double& bx, double& by, double& cx, double& cy) {
  ax = 0.0; ay = 0.0; bx = 1.0; by = 0.0; cx = 0.0; cy = 1.0;
  for (int l = d - 1; l >= 0; --l) {
    const int ch = (int)((path >> (2 * l)) & 3ull);
    const double abx = (ax + bx) * 0.5, aby = (ay + by) * 0.5;
    const double bcx = (bx + cx) * 0.5, bcy = (by + cy) * 0.5;
    const double cax = (cx + ax) * 0.5, cay = (cy + ay) * 0.5;
    if (ch == 0) { bx = abx; by = aby; cx = cax; cy = cay; }
    else if (ch == 1) { ax = abx; ay = aby; cx = bcx; cy = bcy; }
    else if (ch == 2) { ax = cax; ay = cay; bx = bcx; by = bcy; }
    else { ax = bcx; ay = bcy; bx = cax; by = cay; cx = abx; cy = aby; }
  }
}

// decode_path in integer arithmetic: the reference vertices of a depth-d
// sub-simplex are dyadic, (i, j) * 2^-d with 0 <= i, j <= 2^d; midpoints at
// scale 2^-l are sums at scale 2^-(l+1).  The doubles built from them are the
// exact values decode_path computes (its halvings are exact), for a few
// integer adds per level instead of 12 FP64 operations.
__device__ __forceinline__ void decode_path_i(unsigned long long path, int d, double& ax, double& ay,
                                              double& bx, double& by, double& cx, double& cy) {
  int aX = 0, aY = 0, bX = 1, bY = 0, cX = 0, cY = 1;
  for (int l = d - 1; l >= 0; --l) {
    const int ch = (int)((path >> (2 * l)) & 3ull);
    const int abX = aX + bX, abY = aY + bY, bcX = bX + cX, bcY = bY + cY, caX = cX + aX, caY = cY + aY;
    const int AX = aX << 1, AY = aY << 1, BX = bX << 1, BY = bY << 1, CX = cX << 1, CY = cY << 1;
    aX = ch == 0 ? AX : ch == 1 ? abX : ch == 2 ? caX : bcX;
    aY = ch == 0 ? AY : ch == 1 ? abY : ch == 2 ? caY : bcY;
    bX = ch == 0 ? abX : ch == 1 ? BX : ch == 2 ? bcX : caX;
    bY = ch == 0 ? abY : ch == 1 ? BY : ch == 2 ? bcY : caY;
    cX = ch == 0 ? caX : ch == 1 ? bcX : ch == 2 ? CX : abX;
    cY = ch == 0 ? caY : ch == 1 ? bcY : ch == 2 ? CY : abY;
  }
  const double s = ldexp(1.0, -d);
  ax = (double)aX * s; ay = (double)aY * s;
  bx = (double)bX * s; by = (double)bY * s;
  cx = (double)cX * s; cy = (double)cY * s;
}

// acceptance test of one sub-simplex (same operation order as the oracle's
// near_rec): rho_d = rho0n 4^{-d/N_n}; rho_d <= 1 accepts.
constexpr int kBallMaxDepth = 20;  // ball model: accept at this depth (oracle: same)

// g = (rd + 1/rd)/2 depends only on the depth: cached per thread in (gd, gv).
__device__ __forceinline__ bool near_accept(const ElemRec& E, double tx, double ty, double rd,
                                            double ax, double ay, double bx, double by, double cx,
                                            double cy, bool& rle1, int d, double ball_factor,
                                            const double l0[3], int& gd, double& gv) {
  rle1 = false;
  if (ball_factor > 0.0) {
    if (d >= kBallMaxDepth) return true;
    const double vxs[3] = {ax, bx, cx}, vys[3] = {ay, by, cy};
    double px[3], py[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      px[k] = rn_add(E.x0, rn_add(rn_mul(vxs[k], E.e1x), rn_mul(vys[k], E.e2x)));
      py[k] = rn_add(E.y0, rn_add(rn_mul(vxs[k], E.e1y), rn_mul(vys[k], E.e2y)));
    }
    return !rn_ball_test(px[0], py[0], px[1], py[1], px[2], py[2], ball_factor, tx, ty);
  }
  if (!(rd > 1.0)) {
    rle1 = true;
    return true;
  }
  if (d != gd) {
    gd = d;
    gv = rn_mul(rn_add(rd, rn_div(1.0, rd)), 0.5);
  }
  const double g = gv;
  const double vxs[3] = {ax, bx, cx}, vys[3] = {ay, by, cy};
  double dist[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double px = rn_add(E.x0, rn_add(rn_mul(vxs[k], E.e1x), rn_mul(vys[k], E.e2x)));
    const double py = rn_add(E.y0, rn_add(rn_mul(vxs[k], E.e1y), rn_mul(vys[k], E.e2y)));
    dist[k] = rn_dist(tx, ty, px, py);
  }
  // every depth-d sub-simplex is the element's depth-0 image scaled by 2^-d
  // with the same side order: side k has length l0[k] 2^-d exactly
  const double sc = ldexp(1.0, -d);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int k1 = (k + 1) % 3;
    if (rn_add(dist[k], dist[k1]) < rn_mul(g, rn_mul(l0[k], sc))) return false;
  }
  return true;
}

// side lengths of the depth-0 image of the reference simplex (oracle's side_lengths0)
__device__ __forceinline__ void side_lengths0(const ElemRec& E, double l0[3]) {
  const double rx[3] = {0.0, 1.0, 0.0}, ry[3] = {0.0, 0.0, 1.0};
  double px[3], py[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    px[k] = rn_add(E.x0, rn_add(rn_mul(rx[k], E.e1x), rn_mul(ry[k], E.e2x)));
    py[k] = rn_add(E.y0, rn_add(rn_mul(rx[k], E.e1y), rn_mul(ry[k], E.e2y)));
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int k1 = (k + 1) % 3;
    l0[k] = rn_dist(px[k1], py[k1], px[k], py[k]);
  }
}

// Leaves are kept in two CSR arrays: depth <= D (the cached levels, K4b
// k_near_c) and depth > D (k_near_int).  Count pass (FILL = false): counts
// every pair's leaves of both kinds (cnt = total, cntc, cntd), keeps the
// first `cap` codes in scratch[p * cap ..] and lists the pairs that have
// deep leaves (`deep`); pairs with more than `cap` leaves append themselves
// to `over` and are walked again by the fill pass (FILL = true, over
// `plist`), the others are distributed by k_leaves_copy -- one full
// subdivision per pair instead of two.
struct LeafOut {
  int64_t* cntc;
  int64_t* cntd;
  const int64_t* offc;
  const int64_t* offd;
  unsigned long long* leafc;
  unsigned long long* leafd;
  int32_t* deep;
  unsigned* n_deep;
  int D;
  const int32_t* pelem;  // pair -> element, for the cached-leaf tag
};

// Load balance: leaf counts per pair vary from 1 to hundreds, so a thread
// per pair leaves most lanes of a warp idle behind its largest pair.  Each
// warp instead owns a chunk of `chunk` pairs (kLeafChunk; 32 = one pair per
// lane for the few overflow pairs of the fill pass); a lane walks one pair at a
// time (its own DFS; leaf order as described for K4a), and lanes
// whose pair is done take the chunk's next pair (ballot + prefix count: the
// assignment is warp-synchronous, and a pair's outputs do not depend on it).
constexpr int kLeafChunk = 128;
// per-pair leaf scratch of the count pass: pairs with more leaves are walked
// again (k_near_leaves<true>); 256 leaves per pair leaves none over on config 2
// (the scratch is written sparsely, only the leaves that exist)
#ifndef VP_LEAF_SCRATCH_MAX
#define VP_LEAF_SCRATCH_MAX 256
#endif
constexpr int kLeafScratchMax = VP_LEAF_SCRATCH_MAX;
#ifndef VP_LEAVES_MINB
#define VP_LEAVES_MINB 5
#endif
// Pending rejected children of the precise-model walk, one 4-bit mask per
// level 1..kMaxPathDepth in two registers (levels 1-16 in lo, 17-32 in hi):
// the depth-first order of a path-code stack without its local memory.
struct LevelMasks {
  unsigned long long lo = 0, hi = 0;
  __device__ __forceinline__ void set(int l, unsigned m) {
    if (l <= 16) lo |= (unsigned long long)m << (4 * (l - 1));
    else hi |= (unsigned long long)m << (4 * (l - 17));
  }
  __device__ __forceinline__ bool empty() const { return (lo | hi) == 0ull; }
  // deepest level with a pending child and its lowest pending child, cleared
  __device__ __forceinline__ void pop(int& l, int& j) {
    if (hi) {
      const int b = 63 - __clzll((long long)hi);
      l = 17 + b / 4;
      const unsigned nib = (unsigned)(hi >> (4 * (l - 17))) & 15u;
      j = __ffs(nib) - 1;
      hi &= ~(1ull << (4 * (l - 17) + j));
    } else {
      const int b = 63 - __clzll((long long)lo);
      l = 1 + b / 4;
      const unsigned nib = (unsigned)(lo >> (4 * (l - 1))) & 15u;
      j = __ffs(nib) - 1;
      lo &= ~(1ull << (4 * (l - 1) + j));
    }
  }
};
static_assert(kMaxPathDepth <= 32, "LevelMasks holds 32 levels");

template <bool FILL, bool BALL>
__global__ void __launch_bounds__(128, VP_LEAVES_MINB)
    k_near_leaves(int64_t n_pairs, const int32_t* __restrict__ pair_tgt,
                  const int32_t* __restrict__ pair_elem, const double2* __restrict__ txy,
                  const ElemRec* __restrict__ el, const RulesDev* __restrict__ R,
                  int64_t* __restrict__ cnt, LeafOut lo, unsigned long long* __restrict__ stats,
                  int* __restrict__ err, CurvesDev CV, const int32_t* __restrict__ plist,
                  unsigned long long* __restrict__ scratch, int cap, int32_t* __restrict__ over,
                  unsigned* __restrict__ n_over, int chunk) {
  __shared__ double skd[kMaxNearDepth + 2];
  for (int i = threadIdx.x; i < kMaxNearDepth + 2; i += blockDim.x) skd[i] = R->kd[i];
  __syncthreads();
  const double ball_factor = BALL ? R->ball_factor : 0.0;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t c0 = wg * chunk, c1 = min(n_pairs, c0 + chunk);
  unsigned long long rle1 = 0;
  int maxd = 0;
  int64_t cursor = c0;  // warp-uniform: next unassigned pair of the chunk
  bool act = false;
  int64_t p = 0;
  double tx = 0.0, ty = 0.0;
  ElemRec E;
  double l0[3];
  int gd = -1;
  double gv = 0.0;
  // precise model: the node to expand next (path, depth; cd < 0: the root is
  // not tested yet) and the pending rejected children per level
  unsigned long long cpath = 0;
  int cd = -1;
  LevelMasks pend;
  // ball model: a stack of path codes (node-by-node walk, depth <= 20)
  unsigned long long stack[BALL ? 3 * kBallMaxDepth + 4 : 1];
  int sp = 0;
  int64_t n = 0, nc = 0, oc = 0, od = 0;
  while (true) {
    const unsigned wm = __ballot_sync(0xffffffffu, !act);
    if (wm) {
      const int64_t mine = cursor + __popc(wm & lt_mask);
      cursor += __popc(wm);
      if (!act && mine < c1) {
        p = plist ? plist[mine] : mine;
        if (curve_id_of(CV, pair_elem[p]) >= 0) {
          if (!FILL) cnt[p] = lo.cntc[p] = lo.cntd[p] = 0;  // curved element: k_near_curved
        } else {
          const double2 tp = txy[pair_tgt[p]];
          tx = tp.x;
          ty = tp.y;
          E = el[pair_elem[p]];
          side_lengths0(E, l0);
          gd = -1;
          if (BALL) {
            sp = 0;
            stack[sp++] = 0ull;
          } else {
            cpath = 0;
            cd = -1;
            pend = LevelMasks();
          }
          n = nc = 0;
          if (FILL) {
            oc = lo.offc[p];
            od = lo.offd[p];
          }
          act = true;
        }
      }
    }
    if (!__any_sync(0xffffffffu, act)) {
      if (cursor >= c1) break;
      continue;
    }
    if (!act) continue;
    bool bad = false, done = false;
    if (!BALL) {
      // precise model: one step expands a rejected node, testing its four
      // children together.  The children's 12 vertex distances are 6 distinct
      // ones (a, b, c, m_ab, m_bc, m_ca; a shared vertex has the same
      // reference coordinates, hence bit-identical distance), so a child test
      // costs 1.5 square roots instead of 3.  Accepted children are emitted in
      // child order; rejected ones become pending at their level and are
      // expanded depth-first, lowest child first.  The leaf set and every
      // counter are those of near_accept node by node (the oracle's near_rec);
      // the order of a pair's leaves differs from the oracle's recursion (an
      // accepted child is emitted before the subtrees of its rejected lower
      // siblings), which only reorders the per-pair sum.
      if (cd < 0) {  // the root
        double ax, ay, bx, by, cx, cy;
        decode_path_i(0ull, 0, ax, ay, bx, by, cx, cy);
        bool le1;
        if (near_accept(E, tx, ty, rn_mul(E.rho0n, skd[0]), ax, ay, bx, by, cx, cy, le1, 0, 0.0, l0, gd, gv)) {
          if (FILL) {
            if (0 <= lo.D) lo.leafc[oc++] = tag_cached(0ull, pair_elem[p]);
            else lo.leafd[od++] = 0ull;
          } else if (n < cap) {
            scratch[p * cap + n] = 0ull;
          }
          ++n;
          nc += 0 <= lo.D ? 1 : 0;
          rle1 += le1 ? 1ull : 0ull;
          done = true;
        } else {
          cd = 0;
        }
      } else {
        const int d = cd;
        const unsigned long long path = cpath;
        double ax, ay, bx, by, cx, cy;
        decode_path_i(path, d, ax, ay, bx, by, cx, cy);
        const int dc = d + 1;
        const double rd = rn_mul(E.rho0n, skd[dc]);
        const unsigned long long base = ((unsigned long long)dc << 58) | (path << 2);
        bool acc4[4];
        const bool le1 = !(rd > 1.0);
        if (le1) {
          acc4[0] = acc4[1] = acc4[2] = acc4[3] = true;
        } else {
          if (dc != gd) {
            gd = dc;
            gv = rn_mul(rn_add(rd, rn_div(1.0, rd)), 0.5);
          }
          const double sc = ldexp(1.0, -dc);
          double th[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) th[k] = rn_mul(gv, rn_mul(l0[k], sc));
          // reference vertices a, b, c, m_ab, m_bc, m_ca (exact dyadics)
          const double vx[6] = {ax, bx, cx, (ax + bx) * 0.5, (bx + cx) * 0.5, (cx + ax) * 0.5};
          const double vy[6] = {ay, by, cy, (ay + by) * 0.5, (by + cy) * 0.5, (cy + ay) * 0.5};
          double dv[6];
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const double px = rn_add(E.x0, rn_add(rn_mul(vx[k], E.e1x), rn_mul(vy[k], E.e2x)));
            const double py = rn_add(E.y0, rn_add(rn_mul(vx[k], E.e1y), rn_mul(vy[k], E.e2y)));
            dv[k] = rn_dist(tx, ty, px, py);
          }
          // child vertex triples (decode_path order): 0 (a, m_ab, m_ca),
          // 1 (m_ab, b, m_bc), 2 (m_ca, m_bc, c), 3 (m_bc, m_ca, m_ab)
          constexpr int cv[4][3] = {{0, 3, 5}, {3, 1, 4}, {5, 4, 2}, {4, 5, 3}};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            bool in = false;
#pragma unroll
            for (int k = 0; k < 3; ++k) in = in || (rn_add(dv[cv[j][k]], dv[cv[j][(k + 1) % 3]]) < th[k]);
            acc4[j] = !in;
          }
        }
        unsigned rej = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!acc4[j]) {
            rej |= 1u << j;
            continue;
          }
          const unsigned long long cc = base | (unsigned long long)j;
          if (FILL) {
            if (dc <= lo.D) lo.leafc[oc++] = tag_cached(cc, pair_elem[p]);
            else lo.leafd[od++] = cc;
          } else if (n < cap) {
            scratch[p * cap + n] = cc;
          }
          ++n;
          nc += dc <= lo.D ? 1 : 0;
          rle1 += le1 ? 1ull : 0ull;
          maxd = max(maxd, dc);
        }
        if (rej) {
          if (dc + 1 > kMaxPathDepth) bad = true;  // excluded on the host (vp_set_rules)
          else pend.set(dc, rej);
        }
        if (!bad) {
          if (pend.empty()) {
            done = true;
          } else {
            int l, j;
            pend.pop(l, j);
            cpath = ((path >> (2 * (dc - l))) << 2) | (unsigned long long)j;
            cd = l;
          }
        }
      }
    } else {
      // ball model: one node of this lane's pair per step
      const unsigned long long code = stack[--sp];
      const int d = (int)(code >> 58);
      const unsigned long long path = code & kPathMask;
      double ax, ay, bx, by, cx, cy;
      decode_path_i(path, d, ax, ay, bx, by, cx, cy);
      bool le1;
      if (near_accept(E, tx, ty, rn_mul(E.rho0n, skd[d]), ax, ay, bx, by, cx, cy, le1, d, ball_factor, l0, gd, gv)) {
        if (FILL) {
          if (d <= lo.D) lo.leafc[oc++] = tag_cached(code, pair_elem[p]);
          else lo.leafd[od++] = code;
        } else if (n < cap) {
          scratch[p * cap + n] = code;
        }
        ++n;
        nc += d <= lo.D ? 1 : 0;
        rle1 += le1 ? 1ull : 0ull;
        maxd = max(maxd, d);
      } else if (d + 1 > kBallMaxDepth) {
        bad = true;
      } else {
        const unsigned long long base = ((unsigned long long)(d + 1) << 58) | (path << 2);
        stack[sp++] = base | 3ull;
        stack[sp++] = base | 2ull;
        stack[sp++] = base | 1ull;
        stack[sp++] = base;
      }
      done = sp == 0;
    }
    if (bad || done) {  // the pair is done
      if (bad) atomicExch(err, 2);
      if (!FILL) {
        if (bad) n = nc = 0;
        cnt[p] = n;
        lo.cntc[p] = nc;
        lo.cntd[p] = n - nc;
        if (n > cap) over[atomicAdd(n_over, 1u)] = (int32_t)p;
        if (n > nc) lo.deep[atomicAdd(lo.n_deep, 1u)] = (int32_t)p;
      }
      act = false;
    }
  }
  if (!FILL) {
    for (int o = 16; o > 0; o >>= 1) {
      rle1 += __shfl_xor_sync(0xffffffffu, rle1, o);
      maxd = max(maxd, __shfl_xor_sync(0xffffffffu, maxd, o));
    }
    if (lane == 0) {
      if (rle1) atomicAdd(&stats[1], rle1);
      atomicMax(&stats[2], (unsigned long long)maxd);
    }
  }
}

// leaves of the pairs that fit the count pass's scratch -> the two CSR arrays
__global__ void k_leaves_copy(int64_t n_pairs, const int64_t* __restrict__ cnt, int cap,
                              const unsigned long long* __restrict__ scratch, LeafOut lo) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int64_t n = cnt[p];
  if (n > cap) return;
  int64_t oc = lo.offc[p], od = lo.offd[p];
  const int32_t e = lo.pelem[p];
  for (int64_t i = 0; i < n; ++i) {
    const unsigned long long code = scratch[p * cap + i];
    if ((int)(code >> 58) <= lo.D) lo.leafc[oc++] = tag_cached(code, e);
    else lo.leafd[od++] = code;
  }
}

// Per-element cache of G = w_i f(xi_{slot,i}) |J_T| 4^-d / (4 pi) at the N_n-rule nodes of every
// sub-simplex of depth <= D (slot = (4^d - 1)/3 + path): a dense
// coefficient-to-value contraction G[e][r] = sum_j Vt[j][r] c_e[j] with the
// host-built Vt[j][r] = w_i K_j(xi_{slot,i}), r = slot * Ln + i.  Each thread
// owns one row r and 8 elements, so Vt is read once per 8 outputs.
constexpr int kCacheNE = 8;
__global__ void __launch_bounds__(256)
    k_near_cache(int64_t E, int M, int64_t R, const double* __restrict__ Vt, const double* __restrict__ coeffs,
                 const ElemRec* __restrict__ el, double* __restrict__ out) {
  __shared__ double sc[kCacheNE][kMaxModes];
  const int64_t e0 = (int64_t)blockIdx.x * kCacheNE;  // x: element chunks (up to 2^31 - 1)
  const int ne = (int)min((int64_t)kCacheNE, E - e0);
  for (int i = threadIdx.x; i < kCacheNE * M; i += blockDim.x) {
    const int k = i / M, j = i - k * M;
    sc[k][j] = k < ne ? coeffs[(e0 + k) * M + j] * el[e0 + k].det : 0.0;  // |J_T| folded in
  }
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (r >= R) return;
  double acc[kCacheNE];
#pragma unroll
  for (int k = 0; k < kCacheNE; ++k) acc[k] = 0.0;
  for (int j = 0; j < M; ++j) {
    const double v = __ldg(Vt + (int64_t)j * R + r);
#pragma unroll
    for (int k = 0; k < kCacheNE; ++k) acc[k] = fma(v, sc[k][j], acc[k]);
  }
#pragma unroll
  for (int k = 0; k < kCacheNE; ++k)
    if (k < ne) out[(e0 + k) * R + r] = acc[k];
}

// The same contraction on the FP64 tensor cores (north_star: DMMA for the
// dense per-triangle coefficient-to-value contraction).  out = A . B with
// A[e][j] = c_e,j |J_e| (E x M) and B = Vt (M x R): a block computes 32
// elements x 64 rows; A and B tiles sit in shared memory with row strides
// = 4 (mod 16) doubles so the m8n8k4 fragment loads are conflict-free; each
// of the 4 warps owns 32 x 16 outputs (4 x 2 DMMA tiles, 16 accumulators).
// K = M padded to a multiple of 4 with zeros.
// elements some pair of this call refers to (the cache is built for them only:
// a rank's shard of a sharded job, the per-pair API's few pairs)
__global__ void k_mark_elems(int64_t n, const int32_t* __restrict__ pelem, uint8_t* __restrict__ used) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) used[pelem[i]] = 1;
}

constexpr int kNcBM = 32, kNcBN = 64;
__host__ __device__ constexpr int nc_stride(int k) { return k + ((4 - k % 16) + 16) % 16; }
__global__ void __launch_bounds__(128)
    k_near_cache_mma(int64_t E, int M, int64_t R, const double* __restrict__ Vt, const double* __restrict__ coeffs,
                     const ElemRec* __restrict__ el, double* __restrict__ out, const uint8_t* __restrict__ used) {
  extern __shared__ __align__(16) double ncs[];
  const int Kp = (M + 3) & ~3;
  const int SA = nc_stride(Kp), SB = nc_stride(kNcBN);
  double* As = ncs;                 // [kNcBM][SA]
  double* Bs = ncs + kNcBM * SA;    // [Kp][SB]
  // 1-D grid, row block fastest: the blocks of one element block run back to
  // back and share its coefficients in L2 (element block fastest re-read all
  // 235 MB of config 4's coefficients once per row block: 28 GB of DRAM reads)
  const int64_t nrb = (R + kNcBN - 1) / kNcBN;
  const int64_t e0 = ((int64_t)blockIdx.x / nrb) * kNcBM;
  const int64_t r0 = ((int64_t)blockIdx.x % nrb) * kNcBN;
  if (used) {  // an element block no pair of the call refers to: nothing to build
    const bool mine = threadIdx.x < kNcBM && e0 + threadIdx.x < E && used[e0 + threadIdx.x];
    if (!__syncthreads_or(mine)) return;
  }
  __shared__ double sdet[kNcBM];
  if (threadIdx.x < kNcBM) sdet[threadIdx.x] = e0 + threadIdx.x < E ? el[e0 + threadIdx.x].det : 0.0;
  __syncthreads();
  for (int i = threadIdx.x; i < kNcBM * Kp; i += blockDim.x) {
    const int m = i / Kp, j = i - m * Kp;
    const int64_t e = e0 + m;
    As[m * SA + j] = (e < E && j < M) ? coeffs[e * M + j] * sdet[m] : 0.0;  // |J_T| folded in
  }
  for (int i = threadIdx.x; i < Kp * kNcBN; i += blockDim.x) {
    const int j = i / kNcBN, n = i - j * kNcBN;
    const int64_t r = r0 + n;
    Bs[j * SB + n] = (j < M && r < R) ? __ldg(Vt + (int64_t)j * R + r) : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  for (int k0 = 0; k0 < Kp; k0 += 4) {
    double a[4], b[2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = As[(mi * 8 + g) * SA + k0 + t];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = Bs[(k0 + t) * SB + w * 16 + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(acc[mi][ni][0]), "+d"(acc[mi][ni][1])
            : "d"(a[mi]), "d"(b[ni]));
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int64_t e = e0 + mi * 8 + g;
    if (e >= E) continue;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int64_t r = r0 + w * 16 + ni * 8 + 2 * t;
      if (r < R) out[e * R + r] = acc[mi][ni][0];
      if (r + 1 < R) out[e * R + r + 1] = acc[mi][ni][1];
    }
  }
}
inline size_t near_cache_mma_smem(int M) {
  const int Kp = (M + 3) & ~3;
  return sizeof(double) * ((size_t)kNcBM * nc_stride(Kp) + (size_t)Kp * nc_stride(kNcBN));
}

// The same GEMM with the tile of V held in shared memory: a block keeps
// V[:, r0 .. r0 + 128) (all M modes of 128 cache rows) and walks kNc2EB
// consecutive 32-element blocks, so V is staged once per 32 tiles instead of
// once per tile and the only per-tile staging is the 32 x M coefficients,
// prefetched one element block ahead with cp.async (two buffers).  A warp owns
// 32 of the 128 rows: 4 x 4 DMMA m8n8k4 tiles, the same k order and the same
// coeffs * det products as k_near_cache_mma, so the cache is bit-identical.
// Row block fastest in the grid: the 33 row blocks of an element chunk run
// together and share its coefficients in L2.
constexpr int kNc2BN = 128, kNc2EB = 32;
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem));
}
__global__ void __launch_bounds__(128)
    k_near_cache_mma2(int64_t E, int M, int64_t R, const double* __restrict__ Vt, const double* __restrict__ coeffs,
                      const ElemRec* __restrict__ el, double* __restrict__ out, const uint8_t* __restrict__ used) {
  extern __shared__ __align__(16) double ncs[];
  const int Kp = (M + 3) & ~3;
  const int SA = nc_stride(Kp), SB = nc_stride(kNc2BN);
  double* Bs = ncs;                      // [Kp][SB]
  double* As0 = ncs + (size_t)Kp * SB;   // two buffers [kNcBM][SA]
  __shared__ double sdet[2][kNcBM];
  const int64_t nrb = (R + kNc2BN - 1) / kNc2BN;
  const int64_t r0 = ((int64_t)blockIdx.x % nrb) * kNc2BN;
  const int64_t nblk_e = (E + kNcBM - 1) / kNcBM;
  const int64_t b0 = ((int64_t)blockIdx.x / nrb) * kNc2EB, b1 = min(b0 + kNc2EB, nblk_e);
  for (int i = threadIdx.x; i < Kp * kNc2BN; i += blockDim.x) {
    const int j = i / kNc2BN, n = i - j * kNc2BN;
    const int64_t r = r0 + n;
    Bs[j * SB + n] = (j < M && r < R) ? __ldg(Vt + (int64_t)j * R + r) : 0.0;
  }
  for (int i = threadIdx.x; i < 2 * kNcBM * SA; i += blockDim.x) As0[i] = 0.0;  // k padding stays zero
  __syncthreads();
  // stage element block b into buffer s: coefficients by cp.async, det by a plain store
  auto stage = [&](int64_t b, int s) {
    double* As = As0 + (size_t)s * kNcBM * SA;
    const int64_t e0 = b * kNcBM;
    const int rows = (int)min((int64_t)kNcBM, E - e0);
    const double* src = coeffs + e0 * M;
    for (int i = threadIdx.x; i < kNcBM * M; i += blockDim.x) {
      const int m = i / M, j = i - m * M;
      if (m < rows) cp_async8(As + m * SA + j, src + i);
      else As[m * SA + j] = 0.0;
    }
    if (threadIdx.x < kNcBM) sdet[s][threadIdx.x] = threadIdx.x < rows ? el[e0 + threadIdx.x].det : 0.0;
    asm volatile("cp.async.commit_group;");
  };
  auto wanted = [&](int64_t b) {  // block-uniform: some element of the block is in the call's pairs
    if (!used) return true;
    const int64_t e0 = b * kNcBM;
    bool any = false;
    for (int m = 0; m < kNcBM && e0 + m < E; ++m) any |= used[e0 + m] != 0;
    return any;
  };
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  int64_t b = b0;
  while (b < b1 && !wanted(b)) ++b;
  if (b < b1) stage(b, 0);
  int s = 0;
  while (b < b1) {
    int64_t bn = b + 1;
    while (bn < b1 && !wanted(bn)) ++bn;
    if (bn < b1) {
      stage(bn, s ^ 1);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncthreads();
    const double* As = As0 + (size_t)s * kNcBM * SA;
    double acc[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    double dt[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) dt[mi] = sdet[s][mi * 8 + g];
    for (int k0 = 0; k0 < Kp; k0 += 4) {
      double a[4], bb[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[(mi * 8 + g) * SA + k0 + t] * dt[mi];  // |J_T| folded in
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bb[ni] = Bs[(k0 + t) * SB + w * 32 + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(acc[mi][ni][0]), "+d"(acc[mi][ni][1])
              : "d"(a[mi]), "d"(bb[ni]));
    }
    const int64_t e0 = b * kNcBM;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int64_t e = e0 + mi * 8 + g;
      if (e >= E) continue;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int64_t r = r0 + w * 32 + ni * 8 + 2 * t;
        if (r < R) out[e * R + r] = acc[mi][ni][0];
        if (r + 1 < R) out[e * R + r + 1] = acc[mi][ni][1];
      }
    }
    __syncthreads();  // the buffer is free for the stage after next
    b = bn;
    s ^= 1;
  }
}
inline size_t near_cache_mma2_smem(int M) {
  const int Kp = (M + 3) & ~3;
  return sizeof(double) * (2 * (size_t)kNcBM * nc_stride(Kp) + (size_t)Kp * nc_stride(kNc2BN));
}

// NPT leaf nodes per call share the density coefficient loads
template <int P, int NPT>
__device__ __forceinline__ double near_nodes(const ShCoef& cc, const double2* __restrict__ ltab,
                                             const double2* a, const double2* ba, const double2* ca,
                                             const double* sc, const double2* nxy, const double* nw,
                                             const bool* valid, double X0, double Y0, double E1x,
                                             double E1y, double E2x, double E2y, double tx, double ty) {
  double xi[NPT], eta[NPT], f[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    xi[i] = fma(nxy[i].y, ca[i].x, fma(nxy[i].x, ba[i].x, a[i].x));
    eta[i] = fma(nxy[i].y, ca[i].y, fma(nxy[i].x, ba[i].y, a[i].y));
  }
  density_n<P, NPT, true>(cc, xi, eta, f);
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const double yx = fma(eta[i], E2x, fma(xi[i], E1x, X0));
    const double yy = fma(eta[i], E2y, fma(xi[i], E1y, Y0));
    const double dx = tx - yx, dy = ty - yy;
    const double v = (nw[i] * sc[i]) * f[i] * fast_log_r2<1>(ltab, fma(dx, dx, dy * dy));
    acc += valid[i] ? v : 0.0;
  }
  return acc;
}

// K4b in two specialisations so each runs at its own occupancy:
//   MODE 0: leaves at depth <= cache_depth (weighted densities read from the
//           per-element cache; ~25 FP64 ops per node) + the element's point
//           sum; writes part_a[p] and part_s[p];
//   MODE 1: deeper leaves (Koornwinder recurrence at every node); writes part_b[p].
// k_near_combine forms corr[p] = part_a + part_b - part_s in fixed order.
template <int P, int MODE>
__global__ void __launch_bounds__(NEAR_WARPS * 32, MODE == 0 ? 4 : VP_NEAR_MINB)
    k_near_int(int64_t n_pairs, const int32_t* __restrict__ pair_tgt, const int32_t* __restrict__ pair_elem,
               const double2* __restrict__ txy, const ElemRec* __restrict__ el,
               const double* __restrict__ coeffs, const int64_t* __restrict__ loff,
               const unsigned long long* __restrict__ leaves, const double* __restrict__ sx,
               const double* __restrict__ sy, const double* __restrict__ sq,
               const RulesDev* __restrict__ R, const double* __restrict__ gcache, int cache_depth,
               double* __restrict__ part, double* __restrict__ part_s, bool exact_zero,
               const int32_t* __restrict__ plist) {
  constexpr int M = (P + 1) * (P + 2) / 2;
  __shared__ double scc[MODE == 1 ? NEAR_WARPS : 1][M];
  __shared__ double2 sga[NEAR_WARPS][32], sgb[NEAR_WARPS][32], sgc[NEAR_WARPS][32];
  __shared__ double sgs[NEAR_WARPS][32];
  __shared__ int sslot[NEAR_WARPS][32];
  __shared__ double2 snxy[kMaxNearRule];
  __shared__ double snw[kMaxNearRule];
  __shared__ double2 sltab[kLogEntries];
  const int Ln = R->len_n, len_q = R->len_q;
  for (int i = threadIdx.x; i < kLogEntries; i += blockDim.x) sltab[i] = g_logtab[i];
  for (int i = threadIdx.x; i < Ln; i += blockDim.x) {
    snxy[i] = make_double2(R->near_x[i], R->near_y[i]);
    snw[i] = R->near_w[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int nslot = cache_depth >= 0 ? ((1 << (2 * (cache_depth + 1))) - 1) / 3 : 0;
  for (int64_t pi_ = (int64_t)blockIdx.x * NEAR_WARPS + wid; pi_ < n_pairs;
       pi_ += (int64_t)gridDim.x * NEAR_WARPS) {
    const int64_t p = plist ? plist[pi_] : pi_;
    const int32_t t = pair_tgt[p], e = pair_elem[p];
    const double2 tp = txy[t];
    const double tx = tp.x, ty = tp.y;
    const ElemRec& Er = el[e];
    const double X0 = Er.x0, Y0 = Er.y0, E1x = Er.e1x, E1y = Er.e1y, E2x = Er.e2x, E2y = Er.e2y;
    const double det = Er.det;
    const int64_t l0 = loff[p], nl = loff[p + 1] - l0;
    const double* gce = gcache + (int64_t)e * nslot * Ln;
    double acc = 0.0;
    bool coeffs_loaded = false;
    for (int64_t lb = 0; lb < nl; lb += 32) {
      const int nb = (int)min((int64_t)32, nl - lb);
      __syncwarp();
      // this mode's leaves of the batch, compacted to the front
      unsigned long long code = 0;
      int d = 0;
      bool mine = false;
      if (lane < nb) {
        code = leaves[l0 + lb + lane];
        d = (int)(code >> 58);
        mine = MODE == 0 ? d <= cache_depth : d > cache_depth;
      }
      const unsigned mm = __ballot_sync(0xffffffffu, mine);
      const int nm = __popc(mm);
      if (nm == 0) continue;
      if (MODE == 1 && !coeffs_loaded) {
        for (int j = lane; j < M; j += 32) scc[MODE == 1 ? wid : 0][j] = coeffs[(int64_t)e * M + j] * c_cn[j];
        coeffs_loaded = true;
      }
      if (mine) {
        const int pos = __popc(mm & lt_mask);
        double ax, ay, bx, by, cx, cy;
        const unsigned long long path = code & kPathMask;
        decode_path(path, d, ax, ay, bx, by, cx, cy);
        sga[wid][pos] = make_double2(ax, ay);
        sgb[wid][pos] = make_double2(bx - ax, by - ay);
        sgc[wid][pos] = make_double2(cx - ax, cy - ay);
        sgs[wid][pos] = det * ldexp(1.0, -2 * d) * kInv4Pi;
        sslot[wid][pos] = ((1 << (2 * d)) - 1) / 3 + (int)path;
      }
      __syncwarp();
      const int total = nm * Ln;
      if constexpr (MODE == 0) {
        int li = lane / Ln, ni = lane - li * Ln;
        for (int j = lane; j < total; j += 32) {
          const double2 a = sga[wid][li], ba = sgb[wid][li], ca = sgc[wid][li], nn = snxy[ni];
          const double xi = fma(nn.y, ca.x, fma(nn.x, ba.x, a.x));
          const double eta = fma(nn.y, ca.y, fma(nn.x, ba.y, a.y));
          const double yx = fma(eta, E2x, fma(xi, E1x, X0));
          const double yy = fma(eta, E2y, fma(xi, E1y, Y0));
          const double dx = tx - yx, dy = ty - yy;
          const double g = __ldg(gce + (int64_t)sslot[wid][li] * Ln + ni);
          acc = fma(sgs[wid][li] * g, fast_log_r2<1>(sltab, fma(dx, dx, dy * dy)), acc);
          ni += 32;
          while (ni >= Ln) { ni -= Ln; ++li; }
        }
      } else {
        // nodes j and j + 32 = (li, ni), (lj, nj); lanes strided by 64
        int li = lane / Ln, ni = lane - li * Ln;
        int lj = (lane + 32) / Ln, nj = lane + 32 - lj * Ln;
        for (int j = lane; j < total; j += 64) {
          const bool ok2 = j + 32 < total;
          const int l2 = ok2 ? lj : li, n2 = ok2 ? nj : ni;
          const double2 ga[2] = {sga[wid][li], sga[wid][l2]}, gb[2] = {sgb[wid][li], sgb[wid][l2]},
                        gc[2] = {sgc[wid][li], sgc[wid][l2]}, nn[2] = {snxy[ni], snxy[n2]};
          const double gs[2] = {sgs[wid][li], sgs[wid][l2]}, nwv[2] = {snw[ni], snw[n2]};
          const bool valid[2] = {true, ok2};
          acc += near_nodes<P, 2>(ShCoef(scc[MODE == 1 ? wid : 0]), sltab, ga, gb, gc, gs, nn, nwv, valid, X0, Y0,
                                  E1x, E1y, E2x, E2y, tx, ty);
          ni += 64;
          while (ni >= Ln) { ni -= Ln; ++li; }
          nj += 64;
          while (nj >= Ln) { nj -= Ln; ++lj; }
        }
      }
    }
    const double val = warp_sum(acc);
    if (lane == 0) part[p] = val;
  }
}

// K4b, cached leaves (depth <= cache_depth): one warp per pair.  Each lane
// owns fixed rule nodes (lane + 32 k), so a node's (u, v) stays in
// registers and the leaf loop is uniform across the warp; per leaf the warp
// reads (broadcast) the physical vectors D0 = t - P_a, BA = P_b - P_a,
// CA = P_c - P_a of the sub-simplex, formed from the slot's reference
// vertices (a per-slot table, no path decoding).  A node then costs
// t - y = D0 - u BA - v CA (4 FMA), r^2 (2), the table log (6 FP64 + I2F)
// and one FMA with the cached G = w f |J_T| 4^-d / (4 pi) (k_near_cache).
// The cache exceeds L2 on large meshes, so each leaf's G values are loaded
// one leaf ahead.  The log table is replicated 8x in dynamic shared memory
// as in K2 (conflict-free quarter-warp loads).  r^2 = 0 cannot occur: a
// near element never contains t and the rule's nodes are interior.  The
// element's point sum (the subtract of subtract-and-add) is k_point_sum.
constexpr int NC_WARPS = 12;
template <int K>  // ceil(len_n / 32) rule nodes per lane
__global__ void __launch_bounds__(NC_WARPS * 32, 2)
    k_near_c(int64_t n_pairs, const int32_t* __restrict__ pair_tgt, const int32_t* __restrict__ pair_elem,
             const double2* __restrict__ txy, const ElemRec* __restrict__ el, const int64_t* __restrict__ loff,
             const unsigned long long* __restrict__ leaves, const RulesDev* __restrict__ R,
             const double* __restrict__ gcache, const double* __restrict__ slot_ref, int cache_depth,
             double* __restrict__ part, unsigned c3ff) {
  extern __shared__ __align__(16) unsigned char nsm[];
  double2* tab = reinterpret_cast<double2*>(nsm);  // kLogEntries x kLogCopies
  __shared__ double4 sD[NC_WARPS][32];
  __shared__ double2 sC[NC_WARPS][32];
  __shared__ int sslot[NC_WARPS][32];
  const int nslot = cache_depth >= 0 ? ((1 << (2 * (cache_depth + 1))) - 1) / 3 : 0;
  for (int i = threadIdx.x; i < kLogEntries * kLogCopies; i += blockDim.x) tab[i] = g_logtab[i / kLogCopies];
  const int Ln = R->len_n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double nu[K], nv[K];
  bool nok[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int n = lane + 32 * k;
    nok[k] = n < Ln;
    nu[k] = nok[k] ? R->near_x[n] : 0.0;
    nv[k] = nok[k] ? R->near_y[n] : 0.0;
  }
  __syncthreads();
  const unsigned laneoff = 16u * (threadIdx.x & (kLogCopies - 1));
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int64_t p = (int64_t)blockIdx.x * NC_WARPS + wid; p < n_pairs; p += (int64_t)gridDim.x * NC_WARPS) {
    const int32_t t = pair_tgt[p], e = pair_elem[p];
    const int64_t l0 = loff[p], nl = loff[p + 1] - l0;
    const double2 tp = txy[t];
    const double tx = tp.x, ty = tp.y;
    const double* gce = gcache + (int64_t)e * nslot * Ln + lane;
    double acc = 0.0;
    for (int64_t lb = 0; lb < nl; lb += 32) {
      const int nb = (int)min((int64_t)32, nl - lb);
      __syncwarp();
      unsigned long long code = 0;
      int d = 0;
      bool mine = false;
      if (lane < nb) {
        code = leaves[l0 + lb + lane];
        d = (int)(code >> 58);
        mine = d <= cache_depth;
      }
      const unsigned mm = __ballot_sync(0xffffffffu, mine);
      const int nm = __popc(mm);
      if (nm == 0) continue;
      if (mine) {
        const ElemRec& Er = el[e];
        const int pos = __popc(mm & lt_mask);
        const int slot = ((1 << (2 * d)) - 1) / 3 + (int)(code & kCPathMask);
        const double* r = slot_ref + 6 * slot;  // a, b - a, c - a of the slot (L1-resident)
        const double pax = fma(r[1], Er.e2x, fma(r[0], Er.e1x, Er.x0));
        const double pay = fma(r[1], Er.e2y, fma(r[0], Er.e1y, Er.y0));
        sD[wid][pos] = make_double4(tx - pax, ty - pay, fma(r[3], Er.e2x, r[2] * Er.e1x),
                                    fma(r[3], Er.e2y, r[2] * Er.e1y));
        sC[wid][pos] = make_double2(fma(r[5], Er.e2x, r[4] * Er.e1x), fma(r[5], Er.e2y, r[4] * Er.e1y));
        sslot[wid][pos] = slot * Ln;
      }
      __syncwarp();
      // cache rows two leaves ahead (the cache exceeds L2 on large meshes)
      double gn[K], gm[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        gn[k] = nok[k] ? __ldg(gce + sslot[wid][0] + 32 * k) : 0.0;
        gm[k] = nok[k] && nm > 1 ? __ldg(gce + sslot[wid][1] + 32 * k) : 0.0;
      }
#pragma unroll 1
      for (int li = 0; li < nm; ++li) {
        double g[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          g[k] = gn[k];
          gn[k] = gm[k];
        }
        if (li + 2 < nm) {
          const int sn = sslot[wid][li + 2];
#pragma unroll
          for (int k = 0; k < K; ++k) gm[k] = nok[k] ? __ldg(gce + sn + 32 * k) : 0.0;
        }
        const double4 dd = sD[wid][li];
        const double2 cc = sC[wid][li];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (k + 1 < K || nok[k]) {
            const double dx = fma(-nu[k], dd.z, fma(-nv[k], cc.x, dd.x));
            const double dy = fma(-nu[k], dd.w, fma(-nv[k], cc.y, dd.y));
            acc = fma(g[k], far_log_r2<false, true>(tab, laneoff, c3ff, fma(dx, dx, dy * dy)), acc);
          }
        }
      }
    }
    const double val = warp_sum(acc);
    if (lane == 0) part[p] = val;
  }
}

// K4b cached leaves, evaluation form: one warp per TARGET.  The cached leaves
// of t's pairs are contiguous in the CSR array, so the warp walks them in
// 32-leaf batches across pair boundaries (a lane finds its leaf's pair among
// t's few pairs); the target and the per-pair index loads are paid once per
// target, not per pair.  Writes the per-target sum part_t[t] (k_assemble adds
// it); the per-pair API keeps k_near_c.
template <int K>
__global__ void __launch_bounds__(NC_WARPS * 32, 2)
    k_near_ct(int64_t T, const int64_t* __restrict__ toff, const int32_t* __restrict__ pair_elem,
              const double2* __restrict__ txy, const ElemRec* __restrict__ el, const int64_t* __restrict__ loff,
              const unsigned long long* __restrict__ leaves, const RulesDev* __restrict__ R,
              const double* __restrict__ gcache, const double* __restrict__ slot_ref, int cache_depth,
              double* __restrict__ part_t, unsigned c3ff) {
  extern __shared__ __align__(16) unsigned char nsm[];
  double2* tab = reinterpret_cast<double2*>(nsm);  // kLogEntries x kLogCopies
  __shared__ double4 sD[NC_WARPS][32];
  __shared__ double2 sC[NC_WARPS][32];
  __shared__ long long sgo[NC_WARPS][32];  // cache row offset of each leaf
  const int nslot = cache_depth >= 0 ? ((1 << (2 * (cache_depth + 1))) - 1) / 3 : 0;
  for (int i = threadIdx.x; i < kLogEntries * kLogCopies; i += blockDim.x) tab[i] = g_logtab[i / kLogCopies];
  const int Ln = R->len_n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double nu[K], nv[K];
  bool nok[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int n = lane + 32 * k;
    nok[k] = n < Ln;
    nu[k] = nok[k] ? R->near_x[n] : 0.0;
    nv[k] = nok[k] ? R->near_y[n] : 0.0;
  }
  __syncthreads();
  const unsigned laneoff = 16u * (threadIdx.x & (kLogCopies - 1));
  const double* gl = gcache + lane;
  for (int64_t t = (int64_t)blockIdx.x * NC_WARPS + wid; t < T; t += (int64_t)gridDim.x * NC_WARPS) {
    const int64_t q0 = toff[t], q1 = toff[t + 1];
    double acc = 0.0;
    if (q1 > q0) {
      const int64_t L0 = loff[q0], L1 = loff[q1];
      const double2 tp = txy[t];
      const double tx = tp.x, ty = tp.y;
      int64_t q = q0;  // this lane's current pair (leaves ascend with the lane's batches)
      for (int64_t lb = L0; lb < L1; lb += 32) {
        const int nb = (int)min((int64_t)32, L1 - lb);
        __syncwarp();
        if (lane < nb) {
          const int64_t Lf = lb + lane;
          while (loff[q + 1] <= Lf) ++q;
          const int32_t e = pair_elem[q];
          const unsigned long long code = leaves[Lf];
          const int d = (int)(code >> 58);
          const ElemRec& Er = el[e];
          const int slot = ((1 << (2 * d)) - 1) / 3 + (int)(code & kCPathMask);
          const double* r = slot_ref + 6 * slot;
          const double pax = fma(r[1], Er.e2x, fma(r[0], Er.e1x, Er.x0));
          const double pay = fma(r[1], Er.e2y, fma(r[0], Er.e1y, Er.y0));
          sD[wid][lane] = make_double4(tx - pax, ty - pay, fma(r[3], Er.e2x, r[2] * Er.e1x),
                                       fma(r[3], Er.e2y, r[2] * Er.e1y));
          sC[wid][lane] = make_double2(fma(r[5], Er.e2x, r[4] * Er.e1x), fma(r[5], Er.e2y, r[4] * Er.e1y));
          sgo[wid][lane] = ((long long)e * nslot + slot) * Ln;
        }
        __syncwarp();
        double gn[K], gm[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          gn[k] = nok[k] ? __ldg(gl + sgo[wid][0] + 32 * k) : 0.0;
          gm[k] = nok[k] && nb > 1 ? __ldg(gl + sgo[wid][1] + 32 * k) : 0.0;
        }
#pragma unroll 1
        for (int li = 0; li < nb; ++li) {
          double g[K];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            g[k] = gn[k];
            gn[k] = gm[k];
          }
          if (li + 2 < nb) {
            const long long sn = sgo[wid][li + 2];
#pragma unroll
            for (int k = 0; k < K; ++k) gm[k] = nok[k] ? __ldg(gl + sn + 32 * k) : 0.0;
          }
          const double4 dd = sD[wid][li];
          const double2 cc = sC[wid][li];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (k + 1 < K || nok[k]) {
              const double dx = fma(-nu[k], dd.z, fma(-nv[k], cc.x, dd.x));
              const double dy = fma(-nu[k], dd.w, fma(-nv[k], cc.y, dd.y));
              acc = fma(g[k], far_log_r2<false, true>(tab, laneoff, c3ff, fma(dx, dx, dy * dy)), acc);
            }
          }
        }
      }
    }
    const double val = warp_sum(acc);
    if (lane == 0) part_t[t] = val;
  }
}

// K4b cached leaves, evaluation form with leaf GROUPS: the warp takes G leaves
// at a time and spreads their G * len_n rule nodes over its 32 * S lane slots
// (slot s = lane + 32 k -> leaf s / len_n, node s % len_n, fixed per lane).
// For the N_n = 12 near rule (49 nodes) G = 3, S = 5 fills 147 of 160 slots
// (92 %; the one-leaf layout of k_near_ct fills 49 of 64) and gives each lane
// S independent log chains per step instead of 2.  A leaf is a row of four
// 16-B fields in shared memory -- D0 = t - P_a, BA, CA and the address of
// its cache row -- stored field-major (row stride 16 B: the batch's writes
// and the reads of adjacent rows are bank-conflict free), so a slot costs one
// address add, four shared loads at immediate offsets and one global load of
// G (loaded a group ahead) besides its 12 FP64 operations.  Rows past the
// batch end are zero geometry with the address of a zero row, so they add
// exactly 0 without a test; the S*32 - G*len_n spare slots (all in slot
// S - 1) are masked.  Summation order per target is fixed (group, slot).
#ifndef VP_NG_WARPS
#define VP_NG_WARPS 8
#endif
#ifndef VP_NG_MINB
#define VP_NG_MINB 2
#endif
constexpr int NG_WARPS = VP_NG_WARPS;
constexpr int kLeafRows = 32 + 4;  // a batch + G - 1 <= 3 zero rows
struct LeafRows {
  double2 d0[NG_WARPS][kLeafRows];
  double2 ba[NG_WARPS][kLeafRows];
  double2 ca[NG_WARPS][kLeafRows];
  ulonglong2 g[NG_WARPS][kLeafRows];  // .x: address of the leaf's cache row
};
constexpr int kOffBA = (int)sizeof(double2) * NG_WARPS * kLeafRows;  // field offsets from d0
constexpr int kOffCA = 2 * kOffBA, kOffG = 3 * kOffBA;
template <int S>
__global__ void __launch_bounds__(NG_WARPS * 32, VP_NG_MINB)
    k_near_cg(int64_t T, const int64_t* __restrict__ toff, const int32_t* __restrict__ pair_elem,
              const double2* __restrict__ txy, const ElemRec* __restrict__ el, const int64_t* __restrict__ loff,
              const unsigned long long* __restrict__ leaves, const RulesDev* __restrict__ R,
              const double* __restrict__ gcache, const double* __restrict__ zrow,
              const double* __restrict__ slot_ref, int cache_depth, int G, double* __restrict__ part_t,
              unsigned c3ff) {
  extern __shared__ __align__(16) unsigned char nsm[];
  double2* tab = reinterpret_cast<double2*>(nsm);  // kLogEntries x kLogCopies
  __shared__ LeafRows sR;
  const int nslot = cache_depth >= 0 ? ((1 << (2 * (cache_depth + 1))) - 1) / 3 : 0;
  for (int i = threadIdx.x; i < kLogEntries * kLogCopies; i += blockDim.x) tab[i] = g_logtab[i / kLogCopies];
  for (int i = threadIdx.x; i < NG_WARPS * kLeafRows; i += blockDim.x) {
    (&sR.d0[0][0])[i] = (&sR.ba[0][0])[i] = (&sR.ca[0][0])[i] = make_double2(0.0, 0.0);
    (&sR.g[0][0])[i] = make_ulonglong2((unsigned long long)zrow, 0ull);
  }
  const int Ln = R->len_n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double nu[S], nv[S];
  int roff[S], noff[S];  // byte offset of the slot's leaf row within a group, rule node
  bool spare = false;    // slot S - 1 beyond the group's nodes
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int s = lane + 32 * k;
    const int lg = s / Ln;
    const bool ok = lg < G;
    if (k == S - 1) spare = !ok;
    roff[k] = ok ? lg * (int)sizeof(double2) : 0;
    noff[k] = ok ? s - lg * Ln : 0;
    nu[k] = ok ? R->near_x[noff[k]] : 0.0;
    nv[k] = ok ? R->near_y[noff[k]] : 0.0;
  }
  __syncthreads();
  const unsigned laneoff = 16u * (threadIdx.x & (kLogCopies - 1));
  const char* wrow = reinterpret_cast<const char*>(&sR.d0[wid][0]);
  for (int64_t t = (int64_t)blockIdx.x * NG_WARPS + wid; t < T; t += (int64_t)gridDim.x * NG_WARPS) {
    const int64_t q0 = toff[t], q1 = toff[t + 1];
    double acc = 0.0;
    if (q1 > q0) {
      const int64_t L0 = loff[q0], L1 = loff[q1];
      const double2 tp = txy[t];
      const double tx = tp.x, ty = tp.y;
      int64_t q = q0;  // this lane's current pair (leaves ascend with the lane's batches)
      for (int64_t lb = L0; lb < L1; lb += 32) {
        const int nb = (int)min((int64_t)32, L1 - lb);
        __syncwarp();
        if (lane < nb) {
          const int64_t Lf = lb + lane;
          while (loff[q + 1] <= Lf) ++q;
          const int32_t e = pair_elem[q];
          const unsigned long long code = leaves[Lf];
          const int d = (int)(code >> 58);
          const ElemRec& Er = el[e];
          const int slot = ((1 << (2 * d)) - 1) / 3 + (int)(code & kCPathMask);
          const double* r = slot_ref + 6 * slot;
          const double pax = fma(r[1], Er.e2x, fma(r[0], Er.e1x, Er.x0));
          const double pay = fma(r[1], Er.e2y, fma(r[0], Er.e1y, Er.y0));
          sR.d0[wid][lane] = make_double2(tx - pax, ty - pay);
          sR.ba[wid][lane] = make_double2(fma(r[3], Er.e2x, r[2] * Er.e1x), fma(r[3], Er.e2y, r[2] * Er.e1y));
          sR.ca[wid][lane] = make_double2(fma(r[5], Er.e2x, r[4] * Er.e1x), fma(r[5], Er.e2y, r[4] * Er.e1y));
          sR.g[wid][lane] = make_ulonglong2((unsigned long long)(gcache + ((int64_t)e * nslot + slot) * Ln), 0ull);
        } else if (lane < nb + 3) {  // zero rows after the batch (rows 32.. stay zero)
          sR.d0[wid][lane] = sR.ba[wid][lane] = sR.ca[wid][lane] = make_double2(0.0, 0.0);
          sR.g[wid][lane] = make_ulonglong2((unsigned long long)zrow, 0ull);
        }
        __syncwarp();
        double gn[S];
#pragma unroll
        for (int k = 0; k < S; ++k)
          gn[k] = __ldg(*reinterpret_cast<const double* const*>(wrow + roff[k] + kOffG) + noff[k]);
#pragma unroll 1
        for (int li = 0; li < nb; li += G) {
          double g[S];
#pragma unroll
          for (int k = 0; k < S; ++k) g[k] = gn[k];
          if (spare) g[S - 1] = 0.0;
          const char* grp = wrow + li * (int)sizeof(double2);
          if (li + G < nb) {
            const char* nxt = grp + G * (int)sizeof(double2);
#pragma unroll
            for (int k = 0; k < S; ++k)
              gn[k] = __ldg(*reinterpret_cast<const double* const*>(nxt + roff[k] + kOffG) + noff[k]);
          }
#pragma unroll
          for (int k = 0; k < S; ++k) {
            const char* r = grp + roff[k];
            const double2 d0 = *reinterpret_cast<const double2*>(r);
            const double2 ba = *reinterpret_cast<const double2*>(r + kOffBA);
            const double2 ca = *reinterpret_cast<const double2*>(r + kOffCA);
            const double dx = fma(-nu[k], ba.x, fma(-nv[k], ca.x, d0.x));
            const double dy = fma(-nu[k], ba.y, fma(-nv[k], ca.y, d0.y));
            acc = fma(g[k], far_log_r2<false, true>(tab, laneoff, c3ff, fma(dx, dx, dy * dy)), acc);
          }
        }
      }
    }
    const double val = warp_sum(acc);
    if (lane == 0) part_t[t] = val;
  }
}

// K4b cached leaves, evaluation form with 8 LANES PER LEAF: lane l works on
// leaf l / 8 of a group of 4 and on its rule nodes (l mod 8) + 8 k, k < K8 =
// ceil(len_n / 8) (49 nodes: 7 slots, 49 of 56 used, 88 %).  A lane reads its
// leaf's D0 / BA / CA and cache-row address once per group (4 shared loads
// for K8 nodes, against 4 per node in k_near_cg) and the G values of its K8
// nodes (8 consecutive doubles per leaf and slot) a group ahead.  Same zero
// rows past a batch and the same fixed summation order per target.
// W warps per block, two blocks per SM.  The register budget follows from W
// (65536 / (2 * 32 W)): the 7 slots of a 49-node rule need 126 registers
// (W = 8).  The 5 slots of the 33-node rule fit 96 without spills and the
// kernel alone runs faster at W = 10 (20 warps per SM: 43.5 against 46.6 ms
// on config 4; 9, 11 and 12 warps: 49.3, 47.2, 46.5 ms), but beside the FMM
// stream the evaluation is slower with it (250 against 211 ms per step: the
// pair stage stretches to 211 ms), so W stays 8.
template <int W>
struct LeafRowsW {
  double2 d0[W][kLeafRows];
  double2 ba[W][kLeafRows];
  double2 ca[W][kLeafRows];
  ulonglong2 g[W][kLeafRows];  // .x: address of the leaf's cache row
};
template <int K8, int W>
__global__ void __launch_bounds__(W * 32, 2)
    k_near_c8(int64_t T, const int64_t* __restrict__ tl, const int32_t* __restrict__ pair_elem,
              const double2* __restrict__ txy, const ElemRec* __restrict__ el, const int64_t* __restrict__ loff,
              const unsigned long long* __restrict__ leaves, const RulesDev* __restrict__ R,
              const double* __restrict__ gcache, const double* __restrict__ zrow,
              const double* __restrict__ slot_ref, int cache_depth, double* __restrict__ part_t, unsigned c3ff) {
  extern __shared__ __align__(16) unsigned char nsm[];
  double2* tab = reinterpret_cast<double2*>(nsm);  // kLogEntries x kLogCopies
  __shared__ LeafRowsW<W> sR;
  const int nslot = cache_depth >= 0 ? ((1 << (2 * (cache_depth + 1))) - 1) / 3 : 0;
  for (int i = threadIdx.x; i < kLogEntries * kLogCopies; i += blockDim.x) tab[i] = g_logtab[i / kLogCopies];
  for (int i = threadIdx.x; i < W * kLeafRows; i += blockDim.x) {
    (&sR.d0[0][0])[i] = (&sR.ba[0][0])[i] = (&sR.ca[0][0])[i] = make_double2(0.0, 0.0);
    (&sR.g[0][0])[i] = make_ulonglong2((unsigned long long)zrow, 0ull);
  }
  const int Ln = R->len_n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int lg = lane >> 3, n0 = lane & 7;
  double nu[K8], nv[K8];
  bool nok[K8];
#pragma unroll
  for (int k = 0; k < K8; ++k) {
    const int n = n0 + 8 * k;
    nok[k] = n < Ln;
    nu[k] = nok[k] ? R->near_x[n] : 0.0;
    nv[k] = nok[k] ? R->near_y[n] : 0.0;
  }
  __syncthreads();
  const unsigned laneoff = 16u * (threadIdx.x & (kLogCopies - 1));
  // Targets in grid-stride order; target t's cached leaves are
  // [tl[t], tl[t + 1]) (tl[t] = loff[toff[t]], one load deep), and the codes
  // of the next batch are loaded while the current batch computes.
  for (int64_t t = (int64_t)blockIdx.x * W + wid; t < T; t += (int64_t)gridDim.x * W) {
    const int64_t L0 = tl[t], L1 = tl[t + 1];
    double acc = 0.0, acc1 = 0.0;
    if (L1 > L0) {
      const double2 tp = txy[t];
      const double tx = tp.x, ty = tp.y;
      unsigned long long code_n = lane < L1 - L0 ? leaves[L0 + lane] : 0ull;
      for (int64_t lb = L0; lb < L1; lb += 32) {
        const int nb = (int)min((int64_t)32, L1 - lb);
        const unsigned long long code = code_n;
        __syncwarp();
        if (lane < nb) {
          const int32_t e = cached_elem(code);
          const int d = (int)(code >> 58);
          const ElemRec& Er = el[e];
          const int slot = ((1 << (2 * d)) - 1) / 3 + (int)(code & kCPathMask);
          const double* r = slot_ref + 6 * slot;
          const double pax = fma(r[1], Er.e2x, fma(r[0], Er.e1x, Er.x0));
          const double pay = fma(r[1], Er.e2y, fma(r[0], Er.e1y, Er.y0));
          sR.d0[wid][lane] = make_double2(tx - pax, ty - pay);
          sR.ba[wid][lane] = make_double2(fma(r[3], Er.e2x, r[2] * Er.e1x), fma(r[3], Er.e2y, r[2] * Er.e1y));
          sR.ca[wid][lane] = make_double2(fma(r[5], Er.e2x, r[4] * Er.e1x), fma(r[5], Er.e2y, r[4] * Er.e1y));
          sR.g[wid][lane] = make_ulonglong2((unsigned long long)(gcache + ((int64_t)e * nslot + slot) * Ln), 0ull);
        } else if (lane < nb + 4) {  // zero rows after the batch (rows 32.. stay zero)
          sR.d0[wid][lane] = sR.ba[wid][lane] = sR.ca[wid][lane] = make_double2(0.0, 0.0);
          sR.g[wid][lane] = make_ulonglong2((unsigned long long)zrow, 0ull);
        }
        if (lb + 32 + lane < L1) code_n = leaves[lb + 32 + lane];
        __syncwarp();
        double gn[K8];
        {
          const double* gr = reinterpret_cast<const double*>(sR.g[wid][lg].x) + n0;
#pragma unroll
          for (int k = 0; k < K8; ++k) gn[k] = nok[k] ? __ldg(gr + 8 * k) : 0.0;
        }
#pragma unroll 1
        for (int li = 0; li < nb; li += 4) {
          double g[K8];
#pragma unroll
          for (int k = 0; k < K8; ++k) g[k] = gn[k];
          const int row = li + lg;
          const double2 d0 = sR.d0[wid][row], ba = sR.ba[wid][row], ca = sR.ca[wid][row];
          if (li + 4 < nb) {
            const double* gr = reinterpret_cast<const double*>(sR.g[wid][row + 4].x) + n0;
#pragma unroll
            for (int k = 0; k < K8; ++k) gn[k] = nok[k] ? __ldg(gr + 8 * k) : 0.0;
          }
#pragma unroll
          for (int k = 0; k < K8; ++k) {
            // no branch for the last slot's missing nodes (49 = 6 x 8 + 1):
            // there nu = nv = 0 and g = 0, the log of |D0|^2 is finite (also
            // for zero rows: the bit-level log maps 0 to a finite value), so
            // the slot adds exactly 0 and the warp does not diverge.  (Two
            // register sets for g used alternately instead of the copy ran
            // slower: 63.1 vs 55.7 ms on config 4.)
            const double dx = fma(-nu[k], ba.x, fma(-nv[k], ca.x, d0.x));
            const double dy = fma(-nu[k], ba.y, fma(-nv[k], ca.y, d0.y));
            double& a = (k & 1) ? acc1 : acc;  // two chains: K8 DFMAs deep -> K8 / 2
            a = fma(g[k], far_log_r2<false, true>(tab, laneoff, c3ff, fma(dx, dx, dy * dy)), a);
          }
        }
      }
    }
    const double val = warp_sum(acc + acc1);
    if (lane == 0) part_t[t] = val;
  }
}

// tl[t] = loff[toff[t]], t in [0, T]: target t's cached leaves are
// [tl[t], tl[t + 1]) (k_near_c8 reads its ranges one load deep)
__global__ void k_tgt_leafrange(int64_t T, const int64_t* __restrict__ toff, const int64_t* __restrict__ loff,
                                int64_t* __restrict__ tl) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= T) tl[t] = loff[toff[t]];
}

// Point sums of subtract-and-add for the per-pair API: part_s[p] =
// sum_{i in T} q_i log r_{t,i}^2 (coincident pairs exactly 0);
// warp per pair, lanes over T's sources.
constexpr int PS_WARPS = 8;
__global__ void __launch_bounds__(PS_WARPS * 32)
    k_point_sum(int64_t n_pairs, const int32_t* __restrict__ pair_tgt, const int32_t* __restrict__ pair_elem,
                const double2* __restrict__ txy, int len_q, const double* __restrict__ sx,
                const double* __restrict__ sy, const double* __restrict__ sq, double* __restrict__ part_s,
                bool exact_zero) {
  __shared__ double2 sltab[kLogEntries];
  for (int i = threadIdx.x; i < kLogEntries; i += blockDim.x) sltab[i] = g_logtab[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t p = (int64_t)blockIdx.x * PS_WARPS + wid; p < n_pairs; p += (int64_t)gridDim.x * PS_WARPS) {
    const double2 tp = txy[pair_tgt[p]];
    const double sub = warp_point_sum(lane, pair_elem[p], len_q, tp.x, tp.y, sx, sy, sq, sltab, exact_zero);
    if (lane == 0) part_s[p] = sub;
  }
}

// corr = a + b; per-pair API: sub = s
__global__ void k_near_combine(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                               const double* __restrict__ s, double* __restrict__ corr, double* __restrict__ sub_out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  corr[p] = a[p] + b[p];
  if (sub_out) sub_out[p] = s[p];
}

// The evaluation's subtract of subtract-and-add, per
// target: psum[t] = sum over S(t) and N(t) of the elements' point sums
// q_i log r^2.  Warp per target, lanes over the flattened (element, source)
// items, so one reduction serves all of t's pairs.  Coincident pairs take the
// far sum's own no-zero-check log and cancel with it.
// The log table is replicated COPIES times (entry k, copy c at k COPIES + c;
// lane l reads copy l mod COPIES).  One copy has half its shared wavefronts
// bank-conflicted, but the kernel waits on its gathers (long_scoreboard):
// config 4 measured 19.9 / 20.3 / 21.0 / 28.8 ms with 1 / 2 / 4 / 8 copies
// (VP_PSUM_COPIES), so the default is one.
constexpr int PT_WARPS = 8;
template <int COPIES>
__global__ void __launch_bounds__(PT_WARPS * 32)
    k_psum_tgt(int64_t T, const double2* __restrict__ txy, const int32_t* __restrict__ self,
               const int64_t* __restrict__ off, const int32_t* __restrict__ ids, int len_q,
               const double* __restrict__ sx, const double* __restrict__ sy, const double* __restrict__ sq,
               double* __restrict__ psum, int idx32) {
  extern __shared__ __align__(16) double2 ptab[];
  for (int i = threadIdx.x; i < kLogEntries * COPIES; i += blockDim.x) ptab[i] = g_logtab[i / COPIES];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double2* sltab = ptab + (lane & (COPIES - 1));
  // Items (element b of S(t) u N(t), source i) flattened over the lanes, four
  // per lane and pass with every load issued before the logs; the element id
  // comes from lane b of a per-target register list (one coalesced load) and
  // b = j / len_q from a multiply-high (exact for j < 32 * 600, len_q < 600).
  const unsigned magic = (unsigned)((1ull << 32) / (unsigned)len_q + 1ull);
  const unsigned ulen = (unsigned)len_q;
  for (int64_t t = (int64_t)blockIdx.x * PT_WARPS + wid; t < T; t += (int64_t)gridDim.x * PT_WARPS) {
    const double2 tp = txy[t];
    const int32_t se = self[t];
    const int64_t o0 = off[t], nn = off[t + 1] - o0;
    const int hs = se >= 0 ? 1 : 0;
    const int64_t nb = nn + hs;
    double s = 0.0, s1 = 0.0;
    if (nb <= 32 && len_q < 600 && idx32) {
      const int32_t my_e = lane < nb ? (lane < hs ? se : ids[o0 + lane - hs]) : 0;
      const unsigned items = (unsigned)nb * ulen, full = items & ~127u;
      // source index of item j = b len_q + i: k = e_b len_q + i = j + (e_b - b) len_q,
      // 32-bit (idx32: the mesh has fewer than 2^32 sources)
      auto load = [&](unsigned j, double& x, double& y, double& q) {
        const unsigned bb = __umulhi(j, magic);
        const unsigned e = (unsigned)__shfl_sync(0xffffffffu, my_e, (int)bb);
        const unsigned k = (e - bb) * ulen + j;
        x = sx[k];
        y = sy[k];
        q = sq[k];
      };
      auto add = [&](const double* xs, const double* ys, const double* qs) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double dx = tp.x - xs[u], dy = tp.y - ys[u];
          double& a = (u & 1) ? s1 : s;
          a = fma(qs[u], fast_log_r2<COPIES, false>(sltab, fma(dx, dx, dy * dy)), a);
        }
      };
      unsigned j0 = 0;
      for (; j0 < full; j0 += 128) {  // whole passes: no bounds test
        double xs[4], ys[4], qs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) load(j0 + lane + 32 * u, xs[u], ys[u], qs[u]);
        add(xs, ys, qs);
      }
      if (j0 < items) {  // the last, partial pass: idle slots re-read item 0 with q = 0
        double xs[4], ys[4], qs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned j = j0 + lane + 32 * u;
          load(j < items ? j : 0u, xs[u], ys[u], qs[u]);
          qs[u] = j < items ? qs[u] : 0.0;
        }
        add(xs, ys, qs);
      }
    } else {  // long lists (all-near elements): element by element
      for (int64_t b = 0; b < nb; ++b) {
        const int32_t e = b < hs ? se : ids[o0 + b - hs];
        for (int j = lane; j < len_q; j += 32) {
          const int64_t k = (int64_t)e * len_q + j;
          const double dx = tp.x - sx[k], dy = tp.y - sy[k];
          s = fma(sq[k], fast_log_r2<COPIES, false>(sltab, fma(dx, dx, dy * dy)), s);
        }
      }
    }
    s = warp_sum(s + s1);
    if (lane == 0) psum[t] = s;
  }
}

// ---------------------------------------------------------------------------
// K5: self_eval in radius-arc-length coordinates.
constexpr int SELF_WARPS = 4;
// dyadic panels per side: N, M <= log2(L / dmin) + 1 <= 45 since dmin >= h > 1e-13 L
constexpr int kMaxSelfPanels = 128;
// arc-length nodes evaluate the sigma polynomials by Horner in the monomial
// basis of x = 2 sigma - 1 up to this order (conditioning (1+sqrt 2)^p <= 1.2e3);
// the Legendre recurrence above it
constexpr int kSelfHornerMaxP = 8;

struct SelfGeom {
  double Ax, Ay, ABx, ABy, L, h, st;
  double Arx, Ary, BRx, BRy;
  int N, Mr, npan;
  bool degenerate;
};

// The oracle's panel count: the number of halvings n = 0, 1, .. (capped at
// 1100) until x 2^-n < dmin (oracle self_eval's `for (x = st; !(x < dmin); x *= 0.5)`).
// Halving is exact while x stays normal, so for normal positive x >= dmin the
// count follows from the two exponents and one mantissa comparison: with
// n0 = exponent(x) - exponent(dmin), x 2^-n0 has dmin's exponent and is below
// dmin iff its mantissa is; one more halving always is.  Anything else
// (zero, subnormal, non-finite) takes the loop itself.
__device__ __forceinline__ int self_halvings(double x, double dmin) {
  const long long bx = __double_as_longlong(x), bd = __double_as_longlong(dmin);
  const int ex = (int)((bx >> 52) & 0x7ff), ed = (int)((bd >> 52) & 0x7ff);
  if (bx > 0 && bd > 0 && ex > 0 && ed > 0 && ex < 0x7ff && ed < 0x7ff) {
    if (x < dmin) return 0;
    const long long mant = (1ll << 52) - 1;
    const int n0 = ex - ed;
    return min(n0 + ((bx & mant) < (bd & mant) ? 0 : 1), 1100);
  }
  int n = 0;
  for (double y = x; !(y < dmin) && n < 1100; y *= 0.5) ++n;
  return n;
}

__device__ __forceinline__ void self_geom(double tx, double ty, double Ax, double Ay, double Bx,
                                          double By, SelfGeom& G) {
  G.Ax = Ax;
  G.Ay = Ay;
  G.ABx = rn_sub(Bx, Ax);
  G.ABy = rn_sub(By, Ay);
  G.L = rn_sqrt(rn_add(rn_mul(G.ABx, G.ABx), rn_mul(G.ABy, G.ABy)));
  const double vAx = rn_sub(tx, Ax), vAy = rn_sub(ty, Ay);
  const double cr = rn_sub(rn_mul(G.ABx, vAy), rn_mul(G.ABy, vAx));
  G.h = rn_div(fabs(cr), G.L);
  G.degenerate = !(G.h > rn_mul(1e-13, G.L));
  const double sp = rn_div(rn_add(rn_mul(vAx, G.ABx), rn_mul(vAy, G.ABy)), G.L);
  G.st = fmin(fmax(sp, 0.0), G.L);
  const double sl = rn_div(G.st, G.L);
  const double gx = rn_add(Ax, rn_mul(sl, G.ABx)), gy = rn_add(Ay, rn_mul(sl, G.ABy));
  const double dmin = rn_dist(tx, ty, gx, gy);
  const int N = self_halvings(G.st, dmin), Mr = self_halvings(rn_sub(G.L, G.st), dmin);
  G.N = N;
  G.Mr = Mr;
  G.npan = N + Mr + 2;
}

// panel boundary b_i, i = 0 .. N+M+2
// 2^-i for 0 <= i <= 1022, exact (scaling by it is ldexp(x, -i) while the
// result stays normal: here x >= 2^i dmin > 0)
__device__ __forceinline__ double pow2m(int i) { return __longlong_as_double((long long)(1023 - i) << 52); }
__device__ __forceinline__ double self_bnd(const SelfGeom& G, int i) {
  if (i == 0) return 0.0;
  if (i <= G.N) return rn_sub(G.st, i <= 1022 ? G.st * pow2m(i) : ldexp(G.st, -i));
  if (i == G.N + 1) return G.st;
  if (i <= G.N + G.Mr + 1) {
    const int k = G.Mr + 1 - (i - G.N - 1);
    return rn_add(G.st, k <= 1022 ? rn_sub(G.L, G.st) * pow2m(k) : ldexp(rn_sub(G.L, G.st), -k));
  }
  return G.L;
}

// Tensor form of the radial-arc-length quadrature.  On the sub-triangle
// (v, A, B), y(r, sigma) = v + r ((A - v) + sigma (B - A)) (reference
// coordinates), f(y(r, sigma)) is a polynomial of degree <= p in r and in
// sigma.  Its tensor Legendre coefficients A_nk follow exactly from (p+1)^2
// values at Gauss-Legendre points.  The GGQ radial sum of the oracle
//   sum_j w_j r_j (log r0 + log r_j) f(r_j, sigma)
// is linear in f, so it equals sum_n beta_n(sigma) (bt_n log r0 + ct_n) with
// the GGQ-rule moments bt_n = sum_j w_j r_j P_n(2 r_j - 1),
// ct_n = sum_j w_j r_j log r_j P_n(2 r_j - 1) -- the same rule applied to the
// same polynomial, for any p.  Contracting with bt/ct once per sub-triangle
// leaves 2 (p+1)-term Legendre sums per arc-length node instead of N_g + 1
// density evaluations.
struct SelfTab {
  int np;                       // p + 1
  int pad;
  double gx[kMaxPdev + 1];      // Gauss-Legendre nodes on [0,1]
  double PL[(kMaxPdev + 1) * (kMaxPdev + 1)];  // (2n+1) w_a P_n(2 x_a - 1), [n][a]
  double bt[kMaxPdev + 1], ct[kMaxPdev + 1];   // GGQ-rule moments
  double la[kMaxPdev + 1], lb[kMaxPdev + 1];   // Legendre recurrence (2k+1)/(k+1), k/(k+1)
  // sigma-direction transform straight to monomials in x = 2 sigma - 1:
  // PM[j][b] = sum_k [x^j]P_k(x) PL[k][b] (p <= kSelfHornerMaxP: Horner at the nodes)
  double PM[(kMaxPdev + 1) * (kMaxPdev + 1)];
  // f(y(r, sigma)) = F(r, s = r sigma) with F of total degree <= p in (r, s):
  // M = (p+1)(p+2)/2 samples at Fekete-type points (sr, ss) of the triangle
  // 0 <= s <= r <= 1 determine it, and the whole chain grid -> (PL, PM) ->
  // moments is one linear map T2 [2(p+1) x M]: (Eb, Ec) = T2 f(samples).
  double sr[kMaxModes], ss[kMaxModes];
  double T2[2 * (kMaxPdev + 1) * kMaxModes];
};

// f at NPT points from its monomial coefficients about the reference centroid
// (k_mono): (X, Y) = (xi, eta) - c0, coefficient of X^i Y^j at
// mono_off(P, j) + i; Horner in X per power of Y, then in Y.  NPT points
// share every coefficient load.
__host__ __device__ constexpr int mono_off(int P, int j) { return j * (P + 1) - j * (j - 1) / 2; }
template <int P, int NPT, class CC>
__device__ __forceinline__ void density_mono(const CC& cc, const double* X, const double* Y, double* out) {
  double f[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) f[q] = cc[mono_off(P, P)];
#pragma unroll
  for (int j = P - 1; j >= 0; --j) {
    const int oj = mono_off(P, j);
    double r[NPT];
    const double top = cc[oj + P - j];
#pragma unroll
    for (int q = 0; q < NPT; ++q) r[q] = top;
#pragma unroll
    for (int i = P - j - 1; i >= 0; --i) {
      const double ci = cc[oj + i];
#pragma unroll
      for (int q = 0; q < NPT; ++q) r[q] = fma(r[q], X[q], ci);
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q) f[q] = fma(f[q], Y[q], r[q]);
  }
#pragma unroll
  for (int q = 0; q < NPT; ++q) out[q] = f[q];
}

// Per target the warp handles the three sub-triangles together where their
// work is independent: lanes 0-2 form the three side geometries, the
// density samples of all three (3 M points) share one pass of the warp, and
// the 3 x 2(p+1) moment polynomials one more; only the arc-length nodes
// (dyadic panels x Gauss-Legendre) go side by side.
struct SelfSide {
  double Ax, Ay, ABx, ABy, L, h, st, avx, avy, BRx, BRy, invL;
  int N, Mr, npan, degenerate, pad;
};
template <int GS>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = GS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One target per group of GS lanes (GS = 16: two targets per warp, so the
// per-target phases whose width is below 32 -- the three side geometries,
// the panel compaction, the moment contraction -- serve two targets per warp
// instruction).  Every loop has a warp-uniform trip count (the maximum over
// the warp's groups) and per-group predicates, so the warp never diverges
// between groups and full-mask shuffles stay valid.
#ifndef VP_SELF_GS
#define VP_SELF_GS 16
#endif
// lanes per target by order: 8-lane groups keep their per-group arrays within
// the 48 KB of static shared memory up to p = 8
constexpr int self_gs(int p) { return (VP_SELF_GS == 8 && p > 8) ? 16 : VP_SELF_GS; }
template <int P, int GS>
__global__ void __launch_bounds__(SELF_WARPS * 32, VP_SELF_MINB)
    k_self(int64_t n_items, const int32_t* __restrict__ item_tgt, const int32_t* __restrict__ item_elem,
           const double2* __restrict__ txy, const ElemRec* __restrict__ el,
           const double* __restrict__ coeffs, const double* __restrict__ sx,
           const double* __restrict__ sy, const double* __restrict__ sq, const RulesDev* __restrict__ R,
           const SelfTab* __restrict__ ST, double* __restrict__ corr, double* __restrict__ sub_out,
           int64_t* __restrict__ panels_out, unsigned long long* __restrict__ stats, CurvesDev CV,
           const double* __restrict__ mono) {
  static_assert(GS == 8 || GS == 16 || GS == 32, "k_self: 8, 16 or 32 lanes per target");
  constexpr int NG = 32 / GS;             // targets per warp
  constexpr int NGB = SELF_WARPS * NG;    // targets per block
  constexpr int M = (P + 1) * (P + 2) / 2;
  constexpr int NP = P + 1;
  constexpr int M3 = 3 * M;
  constexpr bool kMono = P <= kMonoMaxP;  // density samples from mono (k_mono)
  // density samples per lane and pass over the 3 M points of a target
#ifndef VP_SELF_SNPT_MAX
#define VP_SELF_SNPT_MAX 6
#endif
  // (the fewest passes with at most VP_SELF_SNPT_MAX points per lane, then
  // the fewest points per lane for that many passes)
  constexpr int SNPASS = (M3 + GS * VP_SELF_SNPT_MAX - 1) / (GS * VP_SELF_SNPT_MAX);
  constexpr int SNPT = (M3 + GS * SNPASS - 1) / (GS * SNPASS);
  // panels compacted per chunk (the node loop runs after each chunk); one
  // zero-weight pad entry at index GS
  __shared__ double scc[NGB][M];
  __shared__ double sF[NGB][M3], sE[NGB][3][2 * NP];
  __shared__ double sPa[NGB][GS + 1], sPb[NGB][GS + 1], sPc[NGB][GS + 1];
  __shared__ SelfSide sS[NGB][3];
  constexpr bool kHorner = P <= kSelfHornerMaxP;
  extern __shared__ __align__(16) double sT2[];  // [2 NP][M], dynamic
  __shared__ double ssr[M], sss[M], sla[NP], slb[NP];
  __shared__ double sglx[kMaxGL], sglw[kMaxGL];
  __shared__ double2 sltab[kLogEntries];
  for (int i = threadIdx.x; i < kLogEntries; i += blockDim.x) sltab[i] = g_logtab[i];
  const int NL = R->n_l, len_q = R->len_q;
  for (int i = threadIdx.x; i < NL; i += blockDim.x) {
    sglx[i] = R->gl_x[i];
    sglw[i] = R->gl_w[i];
  }
  for (int i = threadIdx.x; i < 2 * NP * M; i += blockDim.x) sT2[i] = ST->T2[i];
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    ssr[i] = ST->sr[i];
    sss[i] = ST->ss[i];
  }
  for (int i = threadIdx.x; i < NP; i += blockDim.x) {
    sla[i] = ST->la[i];
    slb[i] = ST->lb[i];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gl = lane & (GS - 1), grp = lane / GS;
  const int g = wid * NG + grp;  // the group's slot in the block's shared arrays
  if (gl == 0) {                 // pad panel: weight 0 at the side's middle
    sPa[g][GS] = 0.5;
    sPb[g][GS] = 0.0;
    sPc[g][GS] = 0.0;
  }
  __syncthreads();
  double* cc = scc[g];
  double* F = sF[g];
  unsigned long long my_panels = 0, my_degen = 0;
  for (int64_t base = ((int64_t)blockIdx.x * SELF_WARPS + wid) * NG; base < n_items;
       base += (int64_t)gridDim.x * NGB) {
    const int64_t it = base + grp;
    const bool have = it < n_items;
    const int32_t t = !have ? 0 : (item_tgt ? item_tgt[it] : (int32_t)it);
    const int32_t e_raw = have ? item_elem[it] : -1;
    if (have && e_raw < 0 && gl == 0) {
      corr[it] = 0.0;
      if (sub_out) sub_out[it] = 0.0;
      if (panels_out) panels_out[it] = 0;
    }
    // an inactive group (no item, target outside, curved element: k_self_curved)
    // runs along on element 0 with every side marked empty and writes nothing
    const bool act = e_raw >= 0 && curve_id_of(CV, e_raw) < 0;
    const int32_t e = act ? e_raw : 0;
    const double2 tp = txy[act ? t : 0];
    const double tx = tp.x, ty = tp.y;
    const ElemRec& Er = el[e];
    __syncwarp();
    if constexpr (kMono) {
      for (int j = gl; j < M; j += GS) cc[j] = mono[(int64_t)e * M + j];
    } else {
      for (int j = gl; j < M; j += GS) cc[j] = coeffs[(int64_t)e * M + j] * c_cn[j];
    }
    if (gl < 3) {
      // side (A, B) = (v_k, v_{k+1}); reference corners (0,0), (1,0), (0,1)
      const int k = gl;
      double txi, teta;
      rn_locate(Er, tx, ty, txi, teta);
      const double Ax = k == 0 ? Er.x0 : (k == 1 ? Er.x1 : Er.x2);
      const double Ay = k == 0 ? Er.y0 : (k == 1 ? Er.y1 : Er.y2);
      const double Bx = k == 0 ? Er.x1 : (k == 1 ? Er.x2 : Er.x0);
      const double By = k == 0 ? Er.y1 : (k == 1 ? Er.y2 : Er.y0);
      SelfGeom G;
      self_geom(tx, ty, Ax, Ay, Bx, By, G);
      const double Arx = k == 1 ? 1.0 : 0.0, Ary = k == 2 ? 1.0 : 0.0;
      SelfSide& S = sS[g][k];
      S.Ax = G.Ax; S.Ay = G.Ay; S.ABx = G.ABx; S.ABy = G.ABy; S.L = G.L; S.h = G.h; S.st = G.st;
      S.invL = 1.0 / G.L;
      S.avx = Arx - txi;  // A - v in reference coordinates
      S.avy = Ary - teta;
      S.BRx = (k == 0 ? 1.0 : 0.0) - Arx;
      S.BRy = (k == 1 ? 1.0 : 0.0) - Ary;
      S.N = G.N; S.Mr = G.Mr;
      S.degenerate = G.degenerate ? 1 : 0;
      // panels the node loop visits: none for a degenerate side or an inactive group
      S.npan = (act && !G.degenerate) ? min(G.npan, kMaxSelfPanels) : 0;
    }
    double txi, teta;
    rn_locate(Er, tx, ty, txi, teta);
    if constexpr (kMono) {  // displacements from the centroid of the monomial expansion
      txi -= kMonoC0;
      teta -= kMonoC0;
    }
    __syncwarp();
    // (1) f at the M Fekete-type samples y = v + r (A - v) + s (B - A) of each
    // sub-triangle (f has total degree <= p in (r, s)); the 3 M points of the
    // target, SNPT per lane and pass (degenerate sides are computed and not used)
    for (int i = SNPT * gl; i < M3; i += GS * SNPT) {
      double xs[SNPT], ys[SNPT], f[SNPT];
#pragma unroll
      for (int q = 0; q < SNPT; ++q) {
        const int iq = min(i + q, M3 - 1);
        const int k = iq >= 2 * M ? 2 : (iq >= M ? 1 : 0), sq_ = iq - k * M;
        const SelfSide& S = sS[g][k];
        xs[q] = fma(sss[sq_], S.BRx, fma(ssr[sq_], S.avx, txi));
        ys[q] = fma(sss[sq_], S.BRy, fma(ssr[sq_], S.avy, teta));
      }
      if constexpr (kMono)
        density_mono<P, SNPT>(ShCoef(cc), xs, ys, f);
      else
        density_n<P, SNPT>(ShCoef(cc), xs, ys, f);
#pragma unroll
      for (int q = 0; q < SNPT; ++q)
        if (i + q < M3) F[i + q] = f[q];
    }
    __syncwarp();
    // (2) the sigma polynomials of the GGQ-rule moments per side, (Eb, Ec) =
    // T2 f (Gauss-Legendre grid interpolation, Legendre transforms in r and
    // sigma and the moment contraction, folded on the host)
    for (int o = gl; o < 3 * 2 * NP; o += GS) {
      const int k = o >= 4 * NP ? 2 : (o >= 2 * NP ? 1 : 0), oo = o - k * 2 * NP;
      const double* Fk = F + k * M;
      const double* Tk = sT2 + oo * M;
      // four independent DFMA chains
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int q = 0;
#pragma unroll 2
      for (; q + 4 <= M; q += 4) {
        s0 = fma(Tk[q], Fk[q], s0);
        s1 = fma(Tk[q + 1], Fk[q + 1], s1);
        s2 = fma(Tk[q + 2], Fk[q + 2], s2);
        s3 = fma(Tk[q + 3], Fk[q + 3], s3);
      }
      for (; q < M; ++q) s0 = fma(Tk[q], Fk[q], s0);
      sE[g][k][oo] = (s0 + s1) + (s2 + s3);
    }
    __syncwarp();
    double acc = 0.0;
    long long npan_item = 0;
    if (act && gl == 0)
      my_degen += (unsigned long long)(sS[g][0].degenerate + sS[g][1].degenerate + sS[g][2].degenerate);
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
      const SelfSide& S = sS[g][k];
      SelfGeom G;
      G.Ax = S.Ax; G.Ay = S.Ay; G.ABx = S.ABx; G.ABy = S.ABy; G.L = S.L; G.h = S.h; G.st = S.st;
      G.N = S.N; G.Mr = S.Mr;
      const double* Eb = sE[g][k];
      const double* Ec = Eb + NP;
      const int npan = S.npan;
      int npan_w = npan;  // warp-uniform chunk loop bound
#pragma unroll
      for (int o = 16; o >= GS; o >>= 1) npan_w = max(npan_w, __shfl_xor_sync(0xffffffffu, npan_w, o));
      const double invL = S.invL;
      double eb[NP], ec[NP];
#pragma unroll
      for (int kk = 0; kk < NP; ++kk) {
        eb[kk] = 0.5 * Eb[kk];
        ec[kk] = Ec[kk];
      }
      const double dAx = G.Ax - tx, dAy = G.Ay - ty;
      auto node = [&](int pp, bool ok, double xg, double wg) {
        const int pc = ok ? pp : GS;  // the pad entry for an idle slot
        const double sl = fma(sPb[g][pc], xg, sPa[g][pc]);
        const double ddx = fma(sl, G.ABx, dAx), ddy = fma(sl, G.ABy, dAy);
        const double lg = fast_log_r2<1>(sltab, fma(ddx, ddx, ddy * ddy));
        const double x = fma(2.0, sl, -1.0);
        double ib, ic;
        if constexpr (kHorner) {
          ib = eb[NP - 1];
          ic = ec[NP - 1];
#pragma unroll
          for (int kk = NP - 2; kk >= 0; --kk) {
            ib = fma(ib, x, eb[kk]);
            ic = fma(ic, x, ec[kk]);
          }
        } else {
          double q0 = 1.0, q1 = x;
          ib = eb[0];
          ic = ec[0];
          if (NP > 1) {
            ib = fma(eb[1], q1, ib);
            ic = fma(ec[1], q1, ic);
          }
#pragma unroll
          for (int kk = 1; kk + 1 < NP; ++kk) {
            const double q2 = fma(sla[kk] * x, q1, -slb[kk] * q0);
            ib = fma(eb[kk + 1], q2, ib);
            ic = fma(ec[kk + 1], q2, ic);
            q0 = q1;
            q1 = q2;
          }
        }
        const double v = fma(sPc[g][pc] * wg, fma(lg, ib, ic), acc);
        acc = ok ? v : acc;
      };
      // (3) arc-length nodes: dyadic panels x Gauss-Legendre,
      // in chunks of GS panels: the chunk's non-empty panels are compacted
      // (ballot) into (a, b, c) with sl = s / L = a + b x_gl and node weight
      // c w_gl = (half width) h w_gl
#pragma unroll 1
      for (int i0 = 0; i0 < npan_w; i0 += GS) {
        const int i = i0 + gl;
        const double s0 = i <= npan ? self_bnd(G, i) : 0.0;
        double s1 = __shfl_down_sync(0xffffffffu, s0, 1, GS);
        if (gl == GS - 1) s1 = i + 1 <= npan ? self_bnd(G, i + 1) : 0.0;
        const bool ne = i < npan && s1 > s0;
        const unsigned bal = (__ballot_sync(0xffffffffu, ne) >> (grp * GS)) & (GS == 32 ? 0xffffffffu : ((1u << (GS & 31)) - 1u));
        if (ne) {
          const int pos = __popc(bal & ((1u << gl) - 1u));
          const double half = 0.5 * (s1 - s0);
          sPa[g][pos] = (0.5 * (s0 + s1)) * invL;
          sPb[g][pos] = half * invL;
          sPc[g][pos] = half * G.h;
        }
        const int nne = __popc(bal);
        npan_item += nne;
        int nne_w = nne;
#pragma unroll
        for (int o = 16; o >= GS; o >>= 1) nne_w = max(nne_w, __shfl_xor_sync(0xffffffffu, nne_w, o));
        __syncwarp();
        if (GS == 8 && NL == 16) {  // lane l keeps nodes l and l + 8 of every panel
          const double xg0 = sglx[gl & 7], wg0 = sglw[gl & 7], xg1 = sglx[(gl & 7) + 8], wg1 = sglw[(gl & 7) + 8];
          for (int pp = 0; pp < nne_w; ++pp) {
            node(pp, pp < nne, xg0, wg0);
            node(pp, pp < nne, xg1, wg1);
          }
        } else if (NL == 16) {  // the default N_l: lane l keeps node l mod 16
          const double xg = sglx[gl & 15], wg = sglw[gl & 15];
#ifndef VP_SELF_NODES
#define VP_SELF_NODES 2
#endif
          constexpr int PS = GS >= 16 ? GS / 16 : 1;  // panels side by side in a group
          for (int pp = gl >> 4; pp < nne_w; pp += PS * VP_SELF_NODES) {
#pragma unroll
            for (int u = 0; u < VP_SELF_NODES; ++u) node(pp + PS * u, pp + PS * u < nne, xg, wg);
          }
        } else {
          const int nodes_w = nne_w * NL;
          int pi = gl / NL, gq = gl - pi * NL;
          for (int j = gl; j < nodes_w; j += GS, gq += GS) {
            while (gq >= NL) { gq -= NL; ++pi; }
            node(pi, pi < nne, sglx[gq], sglw[gq]);
          }
        }
        __syncwarp();
      }
    }
    const double val = group_sum<GS>(acc) * kInv2Pi;
    // the evaluation subtracts every point sum of t at once (k_psum_tgt); the
    // per-pair API returns this element's own
    double sub = 0.0;
    if (sub_out) {
      for (int i = gl; i < len_q; i += GS) {
        const int64_t kq = (int64_t)e * len_q + i;
        const double dx = tx - sx[kq], dy = ty - sy[kq];
        sub = fma(sq[kq], fast_log_r2<1, true>(sltab, fma(dx, dx, dy * dy)), sub);
      }
      sub = group_sum<GS>(sub);
    }
    if (act && gl == 0) {
      corr[it] = val;
      if (sub_out) sub_out[it] = sub;
      if (panels_out) panels_out[it] = npan_item;
      my_panels += (unsigned long long)npan_item;
    }
    __syncwarp();
  }
  if (gl == 0 && my_panels) atomicAdd(&stats[3], my_panels);
  if (gl == 0 && my_degen) atomicAdd(&stats[4], my_degen);
}
inline size_t self_dyn_smem(int p) { return sizeof(double) * 2 * (p + 1) * koorn_size(p); }

// ---------------------------------------------------------------------------
// Curved elements (oracle near_rec / self_eval_curved).
// The pairs and self items whose element is curved skip K4/K5 and take these
// kernels: one warp per item, the element's coefficients in shared memory.
//  * k_near_curved: the warp walks the 4-way subdivision depth-first in
//    lockstep (a per-warp stack of path codes in shared memory); acceptance
//    uses the blended sub-simplex vertices and their chords with exact
//    rounding (leaf counts match the oracle); lanes split each leaf's N_n
//    nodes, each weighted by |J| of the blending map.
//  * k_self_curved: sub-elements (t, gamma) and the two straight sides; the
//    density at every (r_j, s) node through the Newton inverse of the
//    blending map seeded on the radial line in reference coordinates.
constexpr int CURV_WARPS = 4;

template <int P>
__global__ void __launch_bounds__(CURV_WARPS * 32)
    k_near_curved(int64_t n_pairs, const int32_t* __restrict__ pair_tgt, const int32_t* __restrict__ pair_elem,
                  const double2* __restrict__ txy, const ElemRec* __restrict__ el,
                  const double* __restrict__ coeffs, CurvesDev CV, const double* __restrict__ sx,
                  const double* __restrict__ sy, const double* __restrict__ sq, const RulesDev* __restrict__ R,
                  double* __restrict__ corr, double* __restrict__ sub_out, int64_t* __restrict__ lcnt,
                  unsigned long long* __restrict__ stats, int* __restrict__ err) {
  constexpr int M = (P + 1) * (P + 2) / 2;
  __shared__ double scc[CURV_WARPS][M];
  __shared__ unsigned long long sstack[CURV_WARPS][kStackCap];
  __shared__ double skd[kMaxNearDepth + 2];
  __shared__ double2 sltab[kLogEntries];
  for (int i = threadIdx.x; i < kLogEntries; i += blockDim.x) sltab[i] = g_logtab[i];
  for (int i = threadIdx.x; i < kMaxNearDepth + 2; i += blockDim.x) skd[i] = R->kd[i];
  __syncthreads();
  const double ball_factor = R->near_model == 1 ? R->ball_factor : 0.0;
  const int Ln = R->len_n, len_q = R->len_q;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long my_leaves = 0, my_rle1 = 0;
  int my_maxd = 0;
  for (int64_t p = (int64_t)blockIdx.x * CURV_WARPS + wid; p < n_pairs; p += (int64_t)gridDim.x * CURV_WARPS) {
    const int32_t e = pair_elem[p];
    const int cid = curve_id_of(CV, e);
    if (cid < 0) continue;
    const CurveRef C = curve_of(CV, cid);
    const ElemRec& Er = el[e];
    const BlendGeom B = bgeom_of(Er);
    const double2 tp = txy[pair_tgt[p]];
    const double tx = tp.x, ty = tp.y;
    __syncwarp();
    for (int j = lane; j < M; j += 32) scc[wid][j] = coeffs[(int64_t)e * M + j] * c_cn[j];
    if (lane == 0) sstack[wid][0] = 0ull;
    __syncwarp();
    int sp = 1;
    bool bad = false;
    double acc = 0.0;
    long long nleaf = 0;
    while (sp > 0) {
      const unsigned long long code = sstack[wid][--sp];
      __syncwarp();
      const int d = (int)(code >> 58);
      const unsigned long long path = code & kPathMask;
      double v[6];
      decode_path(path, d, v[0], v[1], v[2], v[3], v[4], v[5]);
      double px[3], py[3];
#pragma unroll 1
      for (int k = 0; k < 3; ++k) blend<true>(B, C, v[2 * k], v[2 * k + 1], px[k], py[k]);
      bool accept, le1 = false;
      if (ball_factor > 0.0) {
        accept = d >= kBallMaxDepth || !rn_ball_test(px[0], py[0], px[1], py[1], px[2], py[2], ball_factor, tx, ty);
      } else {
        const double rd = rn_mul(Er.rho0n, skd[d]);
        if (!(rd > 1.0)) {
          accept = le1 = true;
        } else {
          const double g = rn_mul(rn_add(rd, rn_div(1.0, rd)), 0.5);
          double dist[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) dist[k] = rn_dist(tx, ty, px[k], py[k]);
          bool nearp = false;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const int k1 = (k + 1) % 3;
            const double len = rn_dist(px[k1], py[k1], px[k], py[k]);
            if (rn_add(dist[k], dist[k1]) < rn_mul(g, len)) nearp = true;
          }
          accept = !nearp;
        }
      }
      if (accept) {
        ++nleaf;
        my_rle1 += le1 ? 1ull : 0ull;
        my_maxd = max(my_maxd, d);
        const double scale = ldexp(1.0, -2 * d) * kInv4Pi;
        const double bax = v[2] - v[0], bay = v[3] - v[1], cax = v[4] - v[0], cay = v[5] - v[1];
        for (int i = lane; i < Ln; i += 32) {
          const double u = R->near_x[i], w = R->near_y[i];
          const double xi = v[0] + (u * bax + w * cax), eta = v[1] + (u * bay + w * cay);
          double yx, yy, J[4];
          blend_jac<false>(B, C, xi, eta, yx, yy, J);
          const double jw = fabs(J[0] * J[3] - J[1] * J[2]);
          const double f = density<P>(ShCoef(scc[wid]), xi, eta);
          const double dx = tx - yx, dy = ty - yy;
          acc += (R->near_w[i] * jw) * f * log(dx * dx + dy * dy) * scale;
        }
      } else {
        if (d + 1 > kMaxPathDepth || sp + 4 > kStackCap) {
          bad = true;
          break;
        }
        const unsigned long long base = ((unsigned long long)(d + 1) << 58) | (path << 2);
        if (lane == 0) {
          sstack[wid][sp] = base | 3ull;
          sstack[wid][sp + 1] = base | 2ull;
          sstack[wid][sp + 2] = base | 1ull;
          sstack[wid][sp + 3] = base;
        }
        sp += 4;
        __syncwarp();
      }
    }
    const double val = warp_sum(acc);
    const double sub = sub_out ? warp_point_sum(lane, e, len_q, tx, ty, sx, sy, sq, sltab, true) : 0.0;
    if (lane == 0) {
      corr[p] = val;
      if (sub_out) sub_out[p] = sub;
      if (lcnt) lcnt[p] = bad ? 0 : nleaf;
      if (bad) atomicExch(err, 2);
      my_leaves += (unsigned long long)nleaf;
    }
  }
  if (lane == 0) {
    if (my_leaves) atomicAdd(&stats[6], my_leaves);
    if (my_rle1) atomicAdd(&stats[1], my_rle1);
    if (my_maxd) atomicMax(&stats[2], (unsigned long long)my_maxd);
  }
}

template <int P>
__global__ void __launch_bounds__(CURV_WARPS * 32)
    k_self_curved(int64_t n_items, const int32_t* __restrict__ item_tgt, const int32_t* __restrict__ item_elem,
                  const double2* __restrict__ txy, const ElemRec* __restrict__ el,
                  const double* __restrict__ coeffs, CurvesDev CV, const double* __restrict__ sx,
                  const double* __restrict__ sy, const double* __restrict__ sq, const RulesDev* __restrict__ R,
                  double* __restrict__ corr, double* __restrict__ sub_out, int64_t* __restrict__ panels_out,
                  unsigned long long* __restrict__ stats) {
  constexpr int M = (P + 1) * (P + 2) / 2;
  __shared__ double scc[CURV_WARPS][M];
  __shared__ double sglx[kMaxGL], sglw[kMaxGL], sgr[kMaxGGQ], sgw[kMaxGGQ], sglr[kMaxGGQ];
  __shared__ double2 sltab[kLogEntries];
  for (int i = threadIdx.x; i < kLogEntries; i += blockDim.x) sltab[i] = g_logtab[i];
  const int NL = R->n_l, NG = R->n_g1, len_q = R->len_q;
  for (int i = threadIdx.x; i < NL; i += blockDim.x) {
    sglx[i] = R->gl_x[i];
    sglw[i] = R->gl_w[i];
  }
  for (int i = threadIdx.x; i < NG; i += blockDim.x) {
    sgr[i] = R->ggq_r[i];
    sgw[i] = R->ggq_w[i] * R->ggq_r[i];
    sglr[i] = R->ggq_lr[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long my_panels = 0, my_degen = 0;
  for (int64_t it = (int64_t)blockIdx.x * CURV_WARPS + wid; it < n_items; it += (int64_t)gridDim.x * CURV_WARPS) {
    const int32_t t = item_tgt ? item_tgt[it] : (int32_t)it;
    const int32_t e = item_elem[it];
    if (e < 0) continue;
    const int cid = curve_id_of(CV, e);
    if (cid < 0) continue;
    const CurveRef C = curve_of(CV, cid);
    const ElemRec& Er = el[e];
    const BlendGeom B = bgeom_of(Er);
    const double2 tp = txy[t];
    const double tx = tp.x, ty = tp.y;
    double txi, teta;
    rn_locate_curved(Er, C, tx, ty, txi, teta);
    __syncwarp();
    for (int j = lane; j < M; j += 32) scc[wid][j] = coeffs[(int64_t)e * M + j] * c_cn[j];
    __syncwarp();
    double acc = 0.0;
    long long npan_item = 0;
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
      const bool arc = k == 0;
      SelfGeom G;
      double grA_x = 0.0, grA_y = 0.0, grB_x = 0.0, grB_y = 0.0;
      if (arc) {
        G.L = C.L;
        G.st = curved_argmin<true>(C, tx, ty);
        double gx, gy;
        curve_eval<true>(C, rn_sub(1.0, G.st / G.L), gx, gy);
        // t on the arc: the sub-element (t, gamma) keeps its area; panels
        // refine down to 1e-9 L (oracle self_eval_curved)
        double dmin = rn_dist(tx, ty, gx, gy);
        if (!(dmin > rn_mul(1e-13, G.L))) dmin = rn_mul(1e-9, G.L);
        G.degenerate = false;
        int N = 0;
        for (double x = G.st; !(x < dmin) && N < 1100; x *= 0.5) ++N;
        int Mr = 0;
        for (double x = rn_sub(G.L, G.st); !(x < dmin) && Mr < 1100; x *= 0.5) ++Mr;
        G.N = N;
        G.Mr = Mr;
        G.npan = N + Mr + 2;
        G.h = 0.0;
      } else {
        // straight sides (v1, v2) and (v2, v0); reference corners (1,0), (0,1), (0,0)
        const double Ax = k == 1 ? Er.x1 : Er.x2, Ay = k == 1 ? Er.y1 : Er.y2;
        const double Bx = k == 1 ? Er.x2 : Er.x0, By = k == 1 ? Er.y2 : Er.y0;
        self_geom(tx, ty, Ax, Ay, Bx, By, G);
        grA_x = k == 1 ? 1.0 : 0.0;
        grA_y = k == 1 ? 0.0 : 1.0;
        grB_x = 0.0;
        grB_y = k == 1 ? 1.0 : 0.0;
      }
      if (G.degenerate) {
        ++my_degen;
        continue;
      }
      const int nodes = G.npan * NL;
      for (int j = lane; j < nodes; j += 32) {
        const int pi = j / NL, gq = j - pi * NL;
        const double s0 = self_bnd(G, pi), s1 = self_bnd(G, pi + 1);
        if (!(s1 > s0)) continue;
        const double mid = 0.5 * (s0 + s1), half = 0.5 * (s1 - s0);
        const double s = mid + half * sglx[gq];
        const double ws = half * sglw[gq];
        const double sl = s / G.L;
        double px, py, jf, grx, gry;
        if (arc) {
          double g[2], g1[2], g2[2];
          curve_eval_d<false>(C, 1.0 - sl, g, g1, g2);
          px = g[0];
          py = g[1];
          const double tgx = -g1[0] / G.L, tgy = -g1[1] / G.L;
          jf = fabs((px - tx) * tgy - (py - ty) * tgx);
          grx = sl;
          gry = 0.0;
        } else {
          px = G.Ax + sl * G.ABx;
          py = G.Ay + sl * G.ABy;
          jf = G.h;
          grx = grA_x + sl * (grB_x - grA_x);
          gry = grA_y + sl * (grB_y - grA_y);
        }
        const double ddx = px - tx, ddy = py - ty;
        const double lr0 = 0.5 * log(ddx * ddx + ddy * ddy);
        double inner = 0.0;
        // rays from t: the preimage of t + r (p - t) is seeded by extrapolating
        // the previous node's preimage along the ray from (txi, teta)
        double pxi = grx, peta = gry, pr = 1.0;
        for (int jg = NG - 1; jg >= 0; --jg) {
          const double rj = sgr[jg];
          const double yx = tx + rj * (px - tx), yy = ty + rj * (py - ty);
          const double fr = rj / pr;
          double xi = txi + fr * (pxi - txi), eta = teta + fr * (peta - teta);
          blend_inverse_tol(B, C, yx, yy, xi, eta, 1e-11);
          pxi = xi;
          peta = eta;
          pr = rj;
          const double xc = fmin(fmax(xi, 0.0), 1.0);
          const double ec = fmin(fmax(eta, 0.0), 1.0 - xc);
          const double f = density<P>(ShCoef(scc[wid]), xc, ec);
          inner += sgw[jg] * (lr0 + sglr[jg]) * f;
        }
        acc += ws * jf * inner;
      }
      for (int pi = 0; pi < G.npan; ++pi)
        if (self_bnd(G, pi + 1) > self_bnd(G, pi)) ++npan_item;
    }
    const double val = warp_sum(acc) * kInv2Pi;
    // the evaluation subtracts every point sum of t at once (k_psum_tgt); the
    // per-pair API returns this element's own
    const double sub = sub_out ? warp_point_sum(lane, e, len_q, tx, ty, sx, sy, sq, sltab, true) : 0.0;
    if (lane == 0) {
      corr[it] = val;
      if (sub_out) sub_out[it] = sub;
      if (panels_out) panels_out[it] = npan_item;
      my_panels += (unsigned long long)npan_item;
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (my_panels) atomicAdd(&stats[3], my_panels);
    if (my_degen) atomicAdd(&stats[4], my_degen);
  }
}

// ---------------------------------------------------------------------------
// Potential interpolation (rules.hpp:129-170 InterpRule /
// interp_coeffs; SPEC.md:566-569, :592-600 PotentialField / field_eval).
// coeffs[e][j] = sum_k Vinv[j][k] values[e][k]: a batched [M x M] x [M x E]
// contraction with the inverse Koornwinder Vandermonde of the interpolation
// nodes; each thread owns one output row j for 8 elements.
__global__ void __launch_bounds__(128)
    k_interp(int64_t E, int M, const double* __restrict__ Vinv, const double* __restrict__ vals,
             double* __restrict__ out) {
  __shared__ double sv[kCacheNE][kMaxModes];
  const int64_t e0 = (int64_t)blockIdx.x * kCacheNE;
  const int ne = (int)min((int64_t)kCacheNE, E - e0);
  for (int i = threadIdx.x; i < kCacheNE * M; i += blockDim.x) {
    const int k = i / M, j = i - k * M;
    sv[k][j] = k < ne ? vals[(e0 + k) * M + j] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    double acc[kCacheNE];
#pragma unroll
    for (int k = 0; k < kCacheNE; ++k) acc[k] = 0.0;
    for (int kk = 0; kk < M; ++kk) {
      const double v = __ldg(Vinv + (int64_t)j * M + kk);
#pragma unroll
      for (int k = 0; k < kCacheNE; ++k) acc[k] = fma(v, sv[k][kk], acc[k]);
    }
#pragma unroll
    for (int k = 0; k < kCacheNE; ++k)
      if (k < ne) out[(e0 + k) * M + j] = acc[k];
  }
}

// field_eval: locate each point in the interpolation mesh (barycentric, tol
// 1e-12, lowest id; candidates from a uniform grid of triangle bboxes) and
// evaluate the element's Koornwinder expansion at the point's reference
// coordinates.  Points outside every element get NaN and elem = -1.
struct TriBox {
  double x0, y0, i00, i01, i10, i11;
};

__global__ void k_tri_boxes(int64_t E, const double2* __restrict__ v, const int32_t* __restrict__ tri,
                            TriBox* __restrict__ tb, double4* __restrict__ bb) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double2 a = v[tri[3 * e]], b = v[tri[3 * e + 1]], c = v[tri[3 * e + 2]];
  const double e1x = b.x - a.x, e1y = b.y - a.y, e2x = c.x - a.x, e2y = c.y - a.y;
  const double det = e1x * e2y - e2x * e1y;
  tb[e] = TriBox{a.x, a.y, e2y / det, -e2x / det, -e1y / det, e1x / det};
  const double pad = 1e-9 * (fabs(e1x) + fabs(e1y) + fabs(e2x) + fabs(e2y));
  bb[e] = make_double4(fmin(a.x, fmin(b.x, c.x)) - pad, fmin(a.y, fmin(b.y, c.y)) - pad,
                       fmax(a.x, fmax(b.x, c.x)) + pad, fmax(a.y, fmax(b.y, c.y)) + pad);
}

__global__ void k_box_count(int64_t E, const double4* __restrict__ bb, GridDev g, int64_t* __restrict__ cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double4 b = bb[e];
  const int cx0 = cell_coord(b.x, g.x0, g.inv_cs, g.nx), cx1 = cell_coord(b.z, g.x0, g.inv_cs, g.nx);
  const int cy0 = cell_coord(b.y, g.y0, g.inv_cs, g.ny), cy1 = cell_coord(b.w, g.y0, g.inv_cs, g.ny);
  cnt[e] = (int64_t)(cx1 - cx0 + 1) * (cy1 - cy0 + 1);
}

__global__ void k_box_fill(int64_t E, const double4* __restrict__ bb, GridDev g, const int64_t* __restrict__ off,
                           int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const double4 b = bb[e];
  const int cx0 = cell_coord(b.x, g.x0, g.inv_cs, g.nx), cx1 = cell_coord(b.z, g.x0, g.inv_cs, g.nx);
  const int cy0 = cell_coord(b.y, g.y0, g.inv_cs, g.ny), cy1 = cell_coord(b.w, g.y0, g.inv_cs, g.ny);
  int64_t o = off[e];
  for (int cy = cy0; cy <= cy1; ++cy)
    for (int cx = cx0; cx <= cx1; ++cx) {
      keys[o] = cy * g.nx + cx;
      vals[o] = (int32_t)e;
      ++o;
    }
}

template <int P>
__global__ void __launch_bounds__(128)
    k_field_eval(int64_t n, const double2* __restrict__ pts, const TriBox* __restrict__ tb,
                 const double4* __restrict__ bb, GridDev g, const int64_t* __restrict__ cbeg,
                 const int64_t* __restrict__ cend, const int32_t* __restrict__ celems,
                 const double* __restrict__ coeffs, double* __restrict__ out, int32_t* __restrict__ elem_out) {
  constexpr int M = (P + 1) * (P + 2) / 2;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 z = pts[i];
  const double fx = floor(rn_mul(rn_sub(z.x, g.x0), g.inv_cs)), fy = floor(rn_mul(rn_sub(z.y, g.y0), g.inv_cs));
  int32_t found = -1;
  double xi = 0.0, eta = 0.0;
  if (fx >= 0.0 && fy >= 0.0 && fx < (double)g.nx && fy < (double)g.ny) {
    const int c = (int)fy * g.nx + (int)fx;
    for (int64_t k = cbeg[c]; k < cend[c] && found < 0; ++k) {
      const int32_t e = celems[k];
      const double4 b = bb[e];
      if (!(z.x >= b.x && z.x <= b.z && z.y >= b.y && z.y <= b.w)) continue;
      const TriBox T = tb[e];
      const double dx = rn_sub(z.x, T.x0), dy = rn_sub(z.y, T.y0);
      const double a = rn_add(rn_mul(T.i00, dx), rn_mul(T.i01, dy));
      const double bq = rn_add(rn_mul(T.i10, dx), rn_mul(T.i11, dy));
      const double l0 = rn_sub(rn_sub(1.0, a), bq);
      if (a >= -kBaryTol && bq >= -kBaryTol && l0 >= -kBaryTol) {
        found = e;
        xi = fmin(fmax(a, 0.0), 1.0);
        eta = fmin(fmax(bq, 0.0), 1.0 - xi);
      }
    }
  }
  elem_out[i] = found;
  if (found < 0) {
    out[i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double cc[M];
  for (int j = 0; j < M; ++j) cc[j] = coeffs[(int64_t)found * M + j] * c_cn[j];
  out[i] = density<P>(cc, xi, eta);
}

// u = (u_far - psum) + near (cached leaves, per target) + sum of the other
// near values (per pair) + self value
__global__ void k_assemble(int64_t T, const double* __restrict__ ufar, const double* __restrict__ psum,
                           const double* __restrict__ neart, const int64_t* __restrict__ off,
                           const double* __restrict__ corr, const double* __restrict__ corr_self,
                           double* __restrict__ u) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  double s = ufar[t] - psum[t];
  if (off[t + 1] > off[t]) s += neart[t];
  for (int64_t p = off[t]; p < off[t + 1]; ++p) s += corr[p];
  s += corr_self[t];
  u[t] = s;
}

__global__ void k_count_self(int64_t T, const int32_t* __restrict__ self,
                             unsigned long long* __restrict__ stats) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = t < T && self[t] >= 0;
  const unsigned b = __ballot_sync(0xffffffffu, in);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(&stats[5], (unsigned long long)__popc(b));
}

// ---------------------------------------------------------------------------
// host side
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 256));
    if (e == cudaSuccess) cap = std::max<size_t>(bytes, 256);
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

double cn_lookup(int n) {  // SPEC.md:430-438; N < 12 clamped to C_12
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

double w_edge(int len, const double* x, const double* y, const double* w) {  // rules.hpp:44-54
  std::vector<double> d(len);
  for (int i = 0; i < len; ++i) d[i] = std::min({x[i], y[i], (1.0 - x[i] - y[i]) / std::sqrt(2.0)});
  std::vector<double> s = d;
  std::nth_element(s.begin(), s.begin() + s.size() / 2, s.end());
  const double med = s[s.size() / 2];
  double best = 0.0;
  for (int i = 0; i < len; ++i)
    if (d[i] < med) best = std::max(best, w[i]);
  return best;
}

}  // namespace

struct vp_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // mesh
  int64_t n_vert = 0, n_tri = 0;
  std::vector<double> h_vxy;
  std::vector<int32_t> h_tri;
  bool have_mesh = false, have_rules = false, have_density = false, sources_valid = false;
  // rules
  vp_rules rules{};
  std::vector<double> h_rules_store;
  RulesDev h_rd{};
  DevBuf d_rules;
  // elements
  DevBuf d_el, d_bbf;  // element records; near-field bboxes rounded outward to float4
  std::vector<int32_t> h_allnear;
  DevBuf d_allnear;
  GridDev grid{};
  DevBuf d_cbeg, d_cend, d_celems;
  // density
  int p = -1, M = 0;
  DevBuf d_coeffs, d_V;
  DevBuf d_kmon, d_mono;  // p <= kMonoMaxP: basis -> centroid monomials [M x M]; per-element monomials [E x M]
  // sources
  DevBuf d_sx, d_sy, d_sq;
  // per-evaluation scratch
  DevBuf d_txy, d_u, d_ufar, d_part, d_self, d_cnt, d_off, d_ids, d_ptgt, d_corr, d_corr_self,
      d_selfref, d_stats, d_err, d_tmp, d_sub, d_leaves, d_pelem, d_lcnt, d_loff, d_leafcodes;
  int64_t n_leaves_last = 0;
  cudaEvent_t ev[10] = {};
  int last_launches = 0;
  // mesh bounding box (root of the FMM tree)
  double bx0 = 0, by0 = 0, bx1 = 0, by1 = 0;
  // far-field method: 0 direct (K2), 1 FMM
  int far_method = 0, fmm_p = 31, fmm_leaf = 40, fmm_levels = 0, tab_p = -1;
  int64_t fmm_outside = 0;
  int max_near_depth = 0;  // deepest near_eval leaf any element can produce (build_elements)
  int psum_copies = 1;     // log-table copies of k_psum_tgt (VP_PSUM_COPIES: 1, 2, 4, 8)
  bool elems_ok = false;   // the last build_elements succeeded
  // Evaluation plan: the host-side sizes an eager evaluation reads back
  // (list and leaf totals, overflow counts, FMM outside targets).  They depend
  // only on the targets, mesh, rules and models -- never on the density -- so
  // a CUDA graph captured with them (vp_evaluate_graph) replays for any
  // density of the same order with no host round trip.
  struct Plan {
    int64_t n_ids = 0, tot0 = 0, tot1 = 0, fmm_nout = 0;
    unsigned list_nover = 0, leaf_nover = 0, ndeep = 0;
    int leaf_cap = 1;
  } plan;
  bool capture = false;  // inside a stream capture: take sizes from `plan`, no host syncs
  uint64_t gen = 1;      // bumped by every vp_set_* that changes the plan or the launch sequence
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  uint64_t g_gen = 0;
  int64_t g_n = -1;
  const void *g_txy = nullptr, *g_u = nullptr;
  unsigned long long* h_gstats = nullptr;  // pinned: stats + error flags of the last replay
  // multi-GPU (vp_multi.cuh): the library's NCCL communicator, if any
  void* comm = nullptr;
  int comm_world = 0, comm_rank = -1;
  DevBuf d_selftab;
  int selftab_p = -1;
  // near-leaf density cache (depth <= cache_depth sub-simplices), see k_near_cache
  int near_model = 0;
  double ball_factor = 1.5;
  int cache_max_depth = 3, cache_depth = -1;
  int64_t cache_max_bytes = 0;  // 0: min(48 GiB, a quarter of the free device memory)
  DevBuf d_elused;  // near cache: elements referred to by the call's pairs
  DevBuf d_cacheV, d_gcache, d_npa, d_npb, d_nps, d_slotref, d_psum, d_lscratch, d_lover, d_nover;
  DevBuf d_lcntc, d_lcntd, d_loffc, d_loffd, d_leafc, d_leafd, d_ldeep;  // leaves split at the cache depth
  DevBuf d_tl;  // per-target cached-leaf ranges (k_tgt_leafrange)
  DevBuf d_lsc, d_tover, d_ntover;  // list build: count-pass id scratch, overflow targets
  DevBuf d_neart;                   // per-target sums of the cached near leaves (evaluation)
  int64_t leaf_scratch_budget = 16ll << 30;  // max bytes of the count pass's leaf scratch (VP_LEAF_SCRATCH_BYTES)
  int tabs_p = -1;  // p of the density-independent tables (K1's V, near-cache Vt, SelfTab); -1: stale
  int cacheV_depth = -2, cacheV_p = -1;
  DevBuf f_tk, f_tk2, f_tv, f_tord;  // FMM: target leaf keys and the leaf order of the targets
  DevBuf f_active;                  // FMM: boxes holding targets (the downward pass skips the others)
  DevBuf f_tab, f_keys, f_keys2, f_vals, f_idx, f_beg, f_end, f_pxy, f_pq, f_mp, f_lp, f_flag, f_oidx,
      f_otxy, f_ou, f_cnt;
  // far field on its own stream and host thread when it overlaps the near and
  // self stages (FMM); fs is the stream the far-path functions use
  cudaStream_t s2 = nullptr, fs = nullptr;
  cudaStream_t s3 = nullptr, ss = nullptr;  // self + point-sum stream (ss: where launch_self goes)
  std::mutex err_mu;
  DevBuf f_tmp;
  int far_launches = 0;
  // curved (blending-map) elements, SURVEY.md §8(f3)
  int curve_deg = 0;
  std::vector<int32_t> h_ecurve, h_celist;
  std::vector<double> h_ccx, h_ccy, h_clen;
  DevBuf d_ecurve, d_ccx, d_ccy, d_clen, d_celist;
};

namespace {

void vp_comm_release(vp_ctx* c);  // vp_multi.cuh

int set_err(vp_ctx* c, int code, const std::string& m) {
  if (c) {
    std::lock_guard<std::mutex> lk(c->err_mu);
    c->err = m;
  }
  return code;
}

#define CUDA_TRY(ctx, x)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      return set_err(ctx, 3, std::string("cuda: ") + cudaGetErrorString(e_) + " at " #x); \
  } while (0)

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

bool has_curves(const vp_ctx* c) { return !c->h_celist.empty(); }
CurvesDev curves_dev(const vp_ctx* c) {
  CurvesDev cv{};
  if (has_curves(c)) {
    cv.ecurve = c->d_ecurve.as<int32_t>();
    cv.cx = c->d_ccx.as<double>();
    cv.cy = c->d_ccy.as<double>();
    cv.len = c->d_clen.as<double>();
    cv.D = c->curve_deg;
  }
  return cv;
}

// Per-element records on the host with the oracle's operation order
// (oracle/vp_oracle.cpp Setup::init): list predicates stay bit-exact.
int build_elements(vp_ctx* c) {
  const int64_t E = c->n_tri;
  const vp_rules& r = c->rules;
  const double we = w_edge(r.len_q, r.far_x, r.far_y, r.far_w);
  const double wn = w_edge(r.len_n, r.near_x, r.near_y, r.near_w);
  const double cq = cn_lookup(r.q), cnn = cn_lookup(r.n_n);
  std::vector<ElemRec> h(E);
  c->h_allnear.clear();
  c->max_near_depth = 0;
  c->elems_ok = false;
  double gx0 = 1e300, gy0 = 1e300, gx1 = -1e300, gy1 = -1e300;
  std::vector<double> ext;
  ext.reserve(E);
  for (int64_t e = 0; e < E; ++e) {
    ElemRec& R = h[e];
    std::memset(&R, 0, sizeof(R));
    const int32_t* id = &c->h_tri[3 * e];
    double px[3], py[3];
    for (int k = 0; k < 3; ++k) {
      px[k] = c->h_vxy[2 * id[k]];
      py[k] = c->h_vxy[2 * id[k] + 1];
    }
    R.x0 = px[0]; R.y0 = py[0]; R.x1 = px[1]; R.y1 = py[1]; R.x2 = px[2]; R.y2 = py[2];
    R.e1x = px[1] - px[0];
    R.e1y = py[1] - py[0];
    R.e2x = px[2] - px[0];
    R.e2y = py[2] - py[0];
    const double t1 = R.e1x * R.e2y;
    const double t2 = R.e2x * R.e1y;
    R.det = t1 - t2;
    if (!(R.det > 0.0))
      return set_err(c, 1, "set_mesh: triangle " + std::to_string(e) +
                               " not counter-clockwise (invariant: det > 0)");
    R.i00 = R.e2y / R.det;
    R.i01 = -R.e2x / R.det;
    R.i10 = -R.e1y / R.det;
    R.i11 = R.e1x / R.det;
    const double w = we * R.det;
    const double den = r.eps * cq;
    const double rho0 = std::pow(w / den, 1.0 / (double)r.q);
    const double wnn = wn * R.det;
    const double denn = r.eps * cnn;
    R.rho0n = std::pow(wnn / denn, 1.0 / (double)r.n_n);
    if (c->near_model == 0) {
      // near_eval accepts every sub-simplex with rho_d = rho0n 4^{-d/N_n} <= 1
      // (SURVEY.md §9.4), so no leaf is deeper than the first such d.  The
      // path codes hold kMaxPathDepth levels (the oracle errors only past
      // kMaxNearDepth = 40): refuse elements that could need more.
      int dstar = 0;
      while (dstar <= kMaxNearDepth && R.rho0n * c->h_rd.kd[dstar] > 1.0) ++dstar;
      if (dstar > kMaxPathDepth)
        return set_err(c, 2, "set_rules: element " + std::to_string(e) + " could need near_eval depth " +
                                 std::to_string(dstar) + " > " + std::to_string(kMaxPathDepth) +
                                 " (path-code limit; rho0 of the N_n model too large: eps too small for the "
                                 "element size)");
      c->max_near_depth = std::max(c->max_near_depth, dstar);
    }
    if (c->near_model == 1) {  // ball model, same operations as the oracle's ball_of
      const double bxr = px[1] - px[0], byr = py[1] - py[0], cxr = px[2] - px[0], cyr = py[2] - py[0];
      const double t1 = bxr * cyr, t2 = byr * cxr;
      const double d = 2.0 * (t1 - t2);
      const double b2 = bxr * bxr + byr * byr, c2 = cxr * cxr + cyr * cyr;
      const double u1 = cyr * b2, u2 = byr * c2, v1 = bxr * c2, v2 = cxr * b2;
      R.ta0 = (u1 - u2) / d;
      R.ta1 = (v1 - v2) / d;
      const double R2 = R.ta0 * R.ta0 + R.ta1 * R.ta1;
      R.ta2 = (c->ball_factor * c->ball_factor) * R2;
      R.ball = 1.0;
      const double rr = std::sqrt(R.ta2) * (1.0 + 1e-9) + 1e-300;
      const double cxm = px[0] + R.ta0, cym = py[0] + R.ta1;
      R.bx0 = cxm - rr; R.by0 = cym - rr; R.bx1 = cxm + rr; R.by1 = cym + rr;
      gx0 = std::min(gx0, R.bx0); gy0 = std::min(gy0, R.by0);
      gx1 = std::max(gx1, R.bx1); gy1 = std::max(gy1, R.by1);
      ext.push_back(std::max(R.bx1 - R.bx0, R.by1 - R.by0));
      continue;
    }
    if (!(rho0 > 1.0)) {  // SPEC.md:444 all-near
      R.ta0 = R.ta1 = R.ta2 = -1.0;
      c->h_allnear.push_back((int32_t)e);
      continue;
    }
    const double g = (rho0 + 1.0 / rho0) * 0.5;
    double ta[3];
    double lox = 1e300, loy = 1e300, hix = -1e300, hiy = -1e300;
    for (int k = 0; k < 3; ++k) {
      const int k1 = (k + 1) % 3;
      const double dx = px[k1] - px[k], dy = py[k1] - py[k];
      const double len = std::sqrt(dx * dx + dy * dy);
      ta[k] = g * len;
      const double mx = (px[k] + px[k1]) * 0.5, my = (py[k] + py[k1]) * 0.5;
      const double rr = ta[k] * 0.5 * (1.0 + 1e-9) + 1e-300;
      lox = std::min(lox, mx - rr); hix = std::max(hix, mx + rr);
      loy = std::min(loy, my - rr); hiy = std::max(hiy, my + rr);
    }
    if (!c->h_ecurve.empty() && c->h_ecurve[e] >= 0) {  // the element bulges past its chord
      const int cid = c->h_ecurve[e], D = c->curve_deg;
      const CurveRef C{c->h_ccx.data() + (int64_t)cid * (D + 1), c->h_ccy.data() + (int64_t)cid * (D + 1), D,
                       c->h_clen[cid]};
      for (int k = 0; k <= 32; ++k) {
        double gx, gy;
        curve_eval<true>(C, k / 32.0, gx, gy);
        const double pad = 1e-9 * C.L + 1e-300;
        lox = std::min(lox, gx - 0.05 * C.L - pad); hix = std::max(hix, gx + 0.05 * C.L + pad);
        loy = std::min(loy, gy - 0.05 * C.L - pad); hiy = std::max(hiy, gy + 0.05 * C.L + pad);
      }
    }
    R.ta0 = ta[0]; R.ta1 = ta[1]; R.ta2 = ta[2];
    R.bx0 = lox; R.by0 = loy; R.bx1 = hix; R.by1 = hiy;
    gx0 = std::min(gx0, lox); gy0 = std::min(gy0, loy);
    gx1 = std::max(gx1, hix); gy1 = std::max(gy1, hiy);
    ext.push_back(std::max(hix - lox, hiy - loy));
  }
  CUDA_TRY(c, c->d_el.ensure(sizeof(ElemRec) * E));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_el.p, h.data(), sizeof(ElemRec) * E, cudaMemcpyHostToDevice, c->stream));
  {
    auto down = [](double x) {
      float f = (float)x;
      if ((double)f > x) f = std::nextafter(f, -INFINITY);
      return f;
    };
    auto up = [](double x) {
      float f = (float)x;
      if ((double)f < x) f = std::nextafter(f, INFINITY);
      return f;
    };
    std::vector<float4> bf(E);
    for (int64_t e = 0; e < E; ++e) {
      const ElemRec& R = h[e];
      if (R.ball == 0.0 && R.ta0 < 0.0)
        bf[e] = make_float4(-INFINITY, -INFINITY, INFINITY, INFINITY);  // all-near
      else
        bf[e] = make_float4(down(R.bx0), down(R.by0), up(R.bx1), up(R.by1));
    }
    CUDA_TRY(c, c->d_bbf.ensure(sizeof(float4) * E));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_bbf.p, bf.data(), sizeof(float4) * E, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  CUDA_TRY(c, c->d_allnear.ensure(sizeof(int32_t) * (c->h_allnear.size() + 1)));
  if (!c->h_allnear.empty())
    CUDA_TRY(c, cudaMemcpyAsync(c->d_allnear.p, c->h_allnear.data(), sizeof(int32_t) * c->h_allnear.size(),
                                cudaMemcpyHostToDevice, c->stream));
  // uniform grid: cell = median near-field extent, capped at 2^24 cells
  GridDev& G = c->grid;
  if (ext.empty()) {
    G.x0 = G.y0 = 0.0;
    G.cs = 1.0;
    G.nx = G.ny = 1;
  } else {
    std::nth_element(ext.begin(), ext.begin() + ext.size() / 2, ext.end());
    double cs = ext[ext.size() / 2];
    const double W = gx1 - gx0, H = gy1 - gy0;
    if (!(cs > 0.0)) cs = std::max(W, H);
    cs *= kGridScale;
    if (const char* gs = getenv("VP_GRID_SCALE")) {  // A/B switch: cell size in median extents
      const double f = atof(gs);
      if (f > 0.0) cs *= f / kGridScale;
    }
    while ((W / cs + 1) * (H / cs + 1) > double(1 << 24)) cs *= 1.5;
    G.x0 = gx0;
    G.y0 = gy0;
    G.cs = cs;
    G.nx = std::max(1, (int)std::ceil(W / cs));
    G.ny = std::max(1, (int)std::ceil(H / cs));
  }
  G.inv_cs = 1.0 / G.cs;
  const int64_t ncell = (int64_t)G.nx * G.ny;
  // bin on the device: count -> scan -> fill -> stable radix sort by cell
  DevBuf cnt, off, keys, vals, keys2, vals2;
  CUDA_TRY(c, cnt.ensure(sizeof(int64_t) * (E + 1)));
  CUDA_TRY(c, off.ensure(sizeof(int64_t) * (E + 1)));
  k_bin_count<<<nblk(E, 256), 256, 0, c->stream>>>(E, c->d_el.as<ElemRec>(), G, cnt.as<int64_t>());
  CUDA_TRY(c, cudaMemsetAsync(cnt.as<int64_t>() + E, 0, sizeof(int64_t), c->stream));
  size_t tmpb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmpb, cnt.as<int64_t>(), off.as<int64_t>(), E + 1, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceScan::ExclusiveSum(c->d_tmp.p, tmpb, cnt.as<int64_t>(), off.as<int64_t>(), E + 1, c->stream);
  int64_t npairs = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&npairs, off.as<int64_t>() + E, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (npairs > (int64_t)INT32_MAX) return set_err(c, 1, "set_rules: element binning too large");
  CUDA_TRY(c, keys.ensure(sizeof(int32_t) * (npairs + 1)));
  CUDA_TRY(c, vals.ensure(sizeof(int32_t) * (npairs + 1)));
  CUDA_TRY(c, keys2.ensure(sizeof(int32_t) * (npairs + 1)));
  CUDA_TRY(c, c->d_celems.ensure(sizeof(int32_t) * (npairs + 1)));
  k_bin_fill<<<nblk(E, 256), 256, 0, c->stream>>>(E, c->d_el.as<ElemRec>(), G, off.as<int64_t>(),
                                                   keys.as<int32_t>(), vals.as<int32_t>());
  int endbit = 1;
  while ((1ll << endbit) < ncell) ++endbit;
  tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, keys.as<int32_t>(), keys2.as<int32_t>(),
                                  vals.as<int32_t>(), c->d_celems.as<int32_t>(), (int)npairs, 0,
                                  endbit, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceRadixSort::SortPairs(c->d_tmp.p, tmpb, keys.as<int32_t>(), keys2.as<int32_t>(),
                                  vals.as<int32_t>(), c->d_celems.as<int32_t>(), (int)npairs, 0,
                                  endbit, c->stream);
  CUDA_TRY(c, c->d_cbeg.ensure(sizeof(int64_t) * ncell));
  CUDA_TRY(c, c->d_cend.ensure(sizeof(int64_t) * ncell));
  CUDA_TRY(c, cudaMemsetAsync(c->d_cbeg.p, 0, sizeof(int64_t) * ncell, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->d_cend.p, 0, sizeof(int64_t) * ncell, c->stream));
  if (npairs > 0)
    k_cell_ranges<<<nblk(npairs, 256), 256, 0, c->stream>>>(npairs, keys2.as<int32_t>(),
                                                             c->d_cbeg.as<int64_t>(), c->d_cend.as<int64_t>());
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->elems_ok = true;
  return 0;
}

#define VP_DISPATCH_P(p, F, ...)      \
  switch (p) {                        \
    case 0: F<0>(__VA_ARGS__); break;   \
    case 1: F<1>(__VA_ARGS__); break;   \
    case 2: F<2>(__VA_ARGS__); break;   \
    case 3: F<3>(__VA_ARGS__); break;   \
    case 4: F<4>(__VA_ARGS__); break;   \
    case 5: F<5>(__VA_ARGS__); break;   \
    case 6: F<6>(__VA_ARGS__); break;   \
    case 7: F<7>(__VA_ARGS__); break;   \
    case 8: F<8>(__VA_ARGS__); break;   \
    case 9: F<9>(__VA_ARGS__); break;   \
    case 10: F<10>(__VA_ARGS__); break; \
    case 11: F<11>(__VA_ARGS__); break; \
    case 12: F<12>(__VA_ARGS__); break; \
    default: break;                     \
  }

template <int K>
void launch_near_c(vp_ctx* c, int blocks, int64_t n, const int32_t* ptgt, const int32_t* pelem, const double2* txy,
                   const double* gc) {
  k_near_c<K><<<std::max(blocks, 1), NC_WARPS * 32, sizeof(LogTab), c->stream>>>(
      n, ptgt, pelem, txy, c->d_el.as<ElemRec>(), c->d_loffc.as<int64_t>(), c->d_leafc.as<unsigned long long>(),
      c->d_rules.as<RulesDev>(), gc, c->d_slotref.as<double>(), c->cache_depth, c->d_npa.as<double>(), 0x3ff00000u);
}

template <int K>
void launch_near_ct(vp_ctx* c, int64_t T, const int64_t* toff, const int32_t* pelem, const double2* txy,
                    const double* gc) {
  const int blocks = (int)std::min<int64_t>(nblk(T, NC_WARPS), (int64_t)c->sm_count * 16);
  k_near_ct<K><<<std::max(blocks, 1), NC_WARPS * 32, sizeof(LogTab), c->stream>>>(
      T, toff, pelem, txy, c->d_el.as<ElemRec>(), c->d_loffc.as<int64_t>(), c->d_leafc.as<unsigned long long>(),
      c->d_rules.as<RulesDev>(), gc, c->d_slotref.as<double>(), c->cache_depth, c->d_neart.as<double>(),
      0x3ff00000u);
}

// Leaf-group shape of k_near_cg: G leaves over 32*S lane slots, the G in 1..4
// (S <= 5) with the highest slot utilisation G*len_n / (32*S); 0 if len_n > 160.
inline int near_group_shape(int Ln, int* S_out) {
  int bestG = 0, bestS = 0;
  double best = 0.0;
  for (int G = 1; G <= 4; ++G) {
    const int S = (G * Ln + 31) / 32;
    if (S > 5) break;
    const double u = (double)(G * Ln) / (32.0 * S);
    if (u > best + 1e-12) best = u, bestG = G, bestS = S;
  }
  *S_out = bestS;
  return bestG;
}

template <int K8>
void launch_near_c8(vp_ctx* c, int64_t T, const int64_t* toff, const int32_t* pelem, const double2* txy,
                    const double* gc) {
  constexpr int W = 8;  // warps per block (see k_near_c8: 10 is faster alone, slower beside the FMM)
  const int blocks = (int)std::min<int64_t>(nblk(T, W), (int64_t)c->sm_count * 24);
  k_tgt_leafrange<<<nblk(T + 1, 256), 256, 0, c->stream>>>(T, toff, c->d_loffc.as<int64_t>(), c->d_tl.as<int64_t>());
  c->last_launches += 1;
  k_near_c8<K8, W><<<std::max(blocks, 1), W * 32, sizeof(LogTab), c->stream>>>(
      T, c->d_tl.as<int64_t>(), pelem, txy, c->d_el.as<ElemRec>(), c->d_loffc.as<int64_t>(), c->d_leafc.as<unsigned long long>(),
      c->d_rules.as<RulesDev>(), gc, gc + c->n_tri * (int64_t)(((1ll << (2 * (c->cache_depth + 1))) - 1) / 3) *
      c->rules.len_n, c->d_slotref.as<double>(), c->cache_depth, c->d_neart.as<double>(), 0x3ff00000u);
}

template <int S>
void launch_near_cg(vp_ctx* c, int G, int64_t T, const int64_t* toff, const int32_t* pelem, const double2* txy,
                    const double* gc) {
  const int blocks = (int)std::min<int64_t>(nblk(T, NG_WARPS), (int64_t)c->sm_count * 24);
  k_near_cg<S><<<std::max(blocks, 1), NG_WARPS * 32, sizeof(LogTab), c->stream>>>(
      T, toff, pelem, txy, c->d_el.as<ElemRec>(), c->d_loffc.as<int64_t>(), c->d_leafc.as<unsigned long long>(),
      c->d_rules.as<RulesDev>(), gc, gc + c->n_tri * (int64_t)(((1ll << (2 * (c->cache_depth + 1))) - 1) / 3) *
      c->rules.len_n, c->d_slotref.as<double>(), c->cache_depth, G, c->d_neart.as<double>(),
      0x3ff00000u);
}

#define VP_DISPATCH_K(k, F, ...)     \
  switch (k) {                       \
    case 1: F<1>(__VA_ARGS__); break; \
    case 2: F<2>(__VA_ARGS__); break; \
    case 3: F<3>(__VA_ARGS__); break; \
    case 4: F<4>(__VA_ARGS__); break; \
    case 5: F<5>(__VA_ARGS__); break; \
    case 6: F<6>(__VA_ARGS__); break; \
    case 7: F<7>(__VA_ARGS__); break; \
    default: F<8>(__VA_ARGS__); break; \
  }

template <int P>
void launch_near_int(vp_ctx* c, int64_t n, const int32_t* ptgt, const int32_t* pelem, const double2* txy,
                     double* corr, double* sub, int64_t ndeep, int64_t T, const int64_t* toff) {
  const int blocks = (int)std::min<int64_t>(nblk(ndeep, NEAR_WARPS), (int64_t)c->sm_count * 32);
  const double* gc = c->cache_depth >= 0 ? c->d_gcache.as<double>() : nullptr;
  const int cblocks = (int)std::min<int64_t>(nblk(n, NC_WARPS), (int64_t)c->sm_count * 16);
  if (sub)
    k_point_sum<<<(unsigned)std::min<int64_t>(nblk(n, PS_WARPS), (int64_t)c->sm_count * 64), PS_WARPS * 32, 0,
                  c->stream>>>(n, ptgt, pelem, txy, c->rules.len_q, c->d_sx.as<double>(), c->d_sy.as<double>(),
                               c->d_sq.as<double>(), c->d_nps.as<double>(), true);
  if (c->cache_depth >= 0 && toff) {  // evaluation: per-target sums of the cached leaves
    cudaMemsetAsync(c->d_npa.p, 0, sizeof(double) * n, c->stream);
    int S = 0;
    const int G = near_group_shape(c->rules.len_n, &S);
    static const bool force_ct = getenv("VP_NEAR_CT") != nullptr;  // A/B switch: one-leaf layout
    static const bool force_cg = getenv("VP_NEAR_CG") != nullptr;  // A/B switch: leaf-group layout
    const int K8 = (c->rules.len_n + 7) / 8;
    if (K8 <= 8 && !force_ct && !force_cg) {
      VP_DISPATCH_K(K8, launch_near_c8, c, T, toff, pelem, txy, gc);
    } else if (G > 0 && !force_ct) {
      switch (S) {
        case 1: launch_near_cg<1>(c, G, T, toff, pelem, txy, gc); break;
        case 2: launch_near_cg<2>(c, G, T, toff, pelem, txy, gc); break;
        case 3: launch_near_cg<3>(c, G, T, toff, pelem, txy, gc); break;
        case 4: launch_near_cg<4>(c, G, T, toff, pelem, txy, gc); break;
        default: launch_near_cg<5>(c, G, T, toff, pelem, txy, gc); break;
      }
    } else {
      VP_DISPATCH_K((c->rules.len_n + 31) / 32, launch_near_ct, c, T, toff, pelem, txy, gc);
    }
  } else if (c->cache_depth >= 0) {
    VP_DISPATCH_K((c->rules.len_n + 31) / 32, launch_near_c, c, cblocks, n, ptgt, pelem, txy, gc);
  } else {
    cudaMemsetAsync(c->d_npa.p, 0, sizeof(double) * n, c->stream);
  }
  // deep leaves (depth > cache depth) of the listed pairs; the others add 0
  cudaMemsetAsync(c->d_npb.p, 0, sizeof(double) * n, c->stream);
  if (ndeep > 0)
    k_near_int<P, 1><<<std::max(blocks, 1), NEAR_WARPS * 32, 0, c->stream>>>(
        ndeep, ptgt, pelem, txy, c->d_el.as<ElemRec>(), c->d_coeffs.as<double>(), c->d_loffd.as<int64_t>(),
        c->d_leafd.as<unsigned long long>(), c->d_sx.as<double>(), c->d_sy.as<double>(), c->d_sq.as<double>(),
        c->d_rules.as<RulesDev>(), nullptr, -1, c->d_npb.as<double>(), nullptr, sub != nullptr,
        c->d_ldeep.as<int32_t>());
  k_near_combine<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->d_npa.as<double>(), c->d_npb.as<double>(),
                                                     c->d_nps.as<double>(), corr, sub);
}

template <int P>
void launch_near_curved(vp_ctx* c, int64_t n, const int32_t* ptgt, const int32_t* pelem, const double2* txy,
                        double* corr, double* sub) {
  const int blocks = (int)std::min<int64_t>(nblk(n, CURV_WARPS), (int64_t)c->sm_count * 16);
  k_near_curved<P><<<std::max(blocks, 1), CURV_WARPS * 32, 0, c->stream>>>(
      n, ptgt, pelem, txy, c->d_el.as<ElemRec>(), c->d_coeffs.as<double>(), curves_dev(c), c->d_sx.as<double>(),
      c->d_sy.as<double>(), c->d_sq.as<double>(), c->d_rules.as<RulesDev>(), corr, sub, c->d_lcnt.as<int64_t>(),
      c->d_stats.as<unsigned long long>(), c->d_err.as<int>());
}

int build_near_cache(vp_ctx* c, const int32_t* pelem, int64_t n_pairs);
void decide_cache_depth(vp_ctx* c);

// T/toff: the evaluation's targets and pair CSR (cached leaves then summed per
// target into d_neart); nullptr for the per-pair API
int launch_near(vp_ctx* c, int64_t n, const int32_t* ptgt, const int32_t* pelem, const double2* txy,
                double* corr, double* sub, int64_t* leaves_host, int64_t T = 0, const int64_t* toff = nullptr) {
  decide_cache_depth(c);
  CUDA_TRY(c, c->d_lcnt.ensure(sizeof(int64_t) * (n + 1)));
  CUDA_TRY(c, c->d_lcntc.ensure(sizeof(int64_t) * (n + 1)));
  CUDA_TRY(c, c->d_lcntd.ensure(sizeof(int64_t) * (n + 1)));
  CUDA_TRY(c, c->d_loffc.ensure(sizeof(int64_t) * (n + 1)));
  CUDA_TRY(c, c->d_loffd.ensure(sizeof(int64_t) * (n + 1)));
  CUDA_TRY(c, c->d_ldeep.ensure(sizeof(int32_t) * (n + 1)));
  // scratch for the first `cap` leaves of every pair (pairs with more are
  // walked again), within a budget: a quarter of the free device memory, at
  // most leaf_scratch_budget (VP_LEAF_SCRATCH_BYTES, default 16 GiB) beyond
  // what the context already holds; halved until the allocation succeeds
  int cap = c->plan.leaf_cap;
  for (;;) {
    if (c->capture) break;  // the eager run's cap; its scratch is allocated
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
      cudaGetLastError();
      free_b = 0;
    }
    static_cast<void>(total_b);
    int64_t budget = std::min<int64_t>(c->leaf_scratch_budget, (int64_t)(free_b / 4) + (int64_t)c->d_lscratch.cap);
    for (;;) {
      cap = (int)std::max<int64_t>(1, std::min<int64_t>(kLeafScratchMax, (budget / 8) / std::max<int64_t>(n, 1)));
      if (c->d_lscratch.ensure(sizeof(unsigned long long) * (size_t)std::max<int64_t>(n * cap, 1)) == cudaSuccess)
        break;
      cudaGetLastError();
      if (cap == 1) return set_err(c, 3, "near_eval: out of device memory for the leaf scratch");
      budget /= 2;
    }
    c->plan.leaf_cap = cap;
    break;
  }
  CUDA_TRY(c, c->d_lover.ensure(sizeof(int32_t) * (n + 1)));
  CUDA_TRY(c, c->d_nover.ensure(2 * sizeof(unsigned)));
  CUDA_TRY(c, cudaMemsetAsync(c->d_nover.p, 0, 2 * sizeof(unsigned), c->stream));
  LeafOut lo{c->d_lcntc.as<int64_t>(), c->d_lcntd.as<int64_t>(), c->d_loffc.as<int64_t>(), c->d_loffd.as<int64_t>(),
             nullptr, nullptr, c->d_ldeep.as<int32_t>(), c->d_nover.as<unsigned>() + 1, c->cache_depth, pelem};
  (c->near_model == 1 ? k_near_leaves<false, true> : k_near_leaves<false, false>)<<<nblk(n, 4 * kLeafChunk), 128, 0,
                                                                                     c->stream>>>(
      n, ptgt, pelem, txy, c->d_el.as<ElemRec>(), c->d_rules.as<RulesDev>(), c->d_lcnt.as<int64_t>(), lo,
      c->d_stats.as<unsigned long long>(), c->d_err.as<int>(), curves_dev(c), nullptr,
      c->d_lscratch.as<unsigned long long>(), cap, c->d_lover.as<int32_t>(), c->d_nover.as<unsigned>(), kLeafChunk);
  CUDA_TRY(c, cudaMemsetAsync(c->d_lcntc.as<int64_t>() + n, 0, sizeof(int64_t), c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->d_lcntd.as<int64_t>() + n, 0, sizeof(int64_t), c->stream));
  size_t tmpb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmpb, c->d_lcntc.as<int64_t>(), c->d_loffc.as<int64_t>(), n + 1, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceScan::ExclusiveSum(c->d_tmp.p, tmpb, c->d_lcntc.as<int64_t>(), c->d_loffc.as<int64_t>(), n + 1,
                                c->stream);
  cub::DeviceScan::ExclusiveSum(c->d_tmp.p, tmpb, c->d_lcntd.as<int64_t>(), c->d_loffd.as<int64_t>(), n + 1,
                                c->stream);
  int64_t tot[2] = {0, 0};
  unsigned nov[2] = {0, 0};
  if (c->capture) {
    tot[0] = c->plan.tot0;
    tot[1] = c->plan.tot1;
    nov[0] = c->plan.leaf_nover;
    nov[1] = c->plan.ndeep;
  } else {
    CUDA_TRY(c, cudaMemcpyAsync(&tot[0], c->d_loffc.as<int64_t>() + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&tot[1], c->d_loffd.as<int64_t>() + n, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(nov, c->d_nover.p, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->plan.tot0 = tot[0];
    c->plan.tot1 = tot[1];
    c->plan.leaf_nover = nov[0];
    c->plan.ndeep = nov[1];
  }
  const int64_t nleaves = tot[0] + tot[1];
  const unsigned nover = nov[0], ndeep = nov[1];
  CUDA_TRY(c, c->d_leafc.ensure(sizeof(unsigned long long) * (tot[0] + 1)));
  CUDA_TRY(c, c->d_leafd.ensure(sizeof(unsigned long long) * (tot[1] + 1)));
  lo.leafc = c->d_leafc.as<unsigned long long>();
  lo.leafd = c->d_leafd.as<unsigned long long>();
  k_leaves_copy<<<nblk(n, 256), 256, 0, c->stream>>>(n, c->d_lcnt.as<int64_t>(), cap,
                                                     c->d_lscratch.as<unsigned long long>(), lo);
  if (nover > 0)
    (c->near_model == 1 ? k_near_leaves<true, true> : k_near_leaves<true, false>)<<<nblk(nover, 128), 128, 0,
                                                                                   c->stream>>>(
        nover, ptgt, pelem, txy, c->d_el.as<ElemRec>(), c->d_rules.as<RulesDev>(), nullptr, lo,
        c->d_stats.as<unsigned long long>(), c->d_err.as<int>(), curves_dev(c), c->d_lover.as<int32_t>(), nullptr, 0,
        nullptr, nullptr, 32);
  if (int rc = build_near_cache(c, pelem, n)) return rc;
  CUDA_TRY(c, c->d_npa.ensure(sizeof(double) * (n + 1)));
  CUDA_TRY(c, c->d_npb.ensure(sizeof(double) * (n + 1)));
  CUDA_TRY(c, c->d_nps.ensure(sizeof(double) * (n + 1)));
  if (toff) {
    CUDA_TRY(c, c->d_neart.ensure(sizeof(double) * (T + 1)));
    CUDA_TRY(c, c->d_tl.ensure(sizeof(int64_t) * (T + 1)));
    if (c->cache_depth < 0) CUDA_TRY(c, cudaMemsetAsync(c->d_neart.p, 0, sizeof(double) * T, c->stream));
  }
  VP_DISPATCH_P(c->p, launch_near_int, c, n, ptgt, pelem, txy, corr, sub, (int64_t)ndeep, T, toff);
  if (has_curves(c)) {
    VP_DISPATCH_P(c->p, launch_near_curved, c, n, ptgt, pelem, txy, corr, sub);
    c->last_launches += 1;
  }
  CUDA_TRY(c, cudaGetLastError());
  c->n_leaves_last = nleaves;
  c->last_launches += 9;
  if (leaves_host)
    CUDA_TRY(c, cudaMemcpyAsync(leaves_host, c->d_lcnt.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
  return 0;
}

template <int P>
void launch_self(vp_ctx* c, int64_t n, const int32_t* itgt, const int32_t* ielem, const double2* txy,
                 double* corr, double* sub, int64_t* panels) {
  const int blocks = (int)std::min<int64_t>(nblk(n, SELF_WARPS * (32 / self_gs(P))), (int64_t)c->sm_count * 64);
  k_self<P, self_gs(P)><<<std::max(blocks, 1), SELF_WARPS * 32, self_dyn_smem(P), c->ss>>>(
      n, itgt, ielem, txy, c->d_el.as<ElemRec>(), c->d_coeffs.as<double>(), c->d_sx.as<double>(),
      c->d_sy.as<double>(), c->d_sq.as<double>(), c->d_rules.as<RulesDev>(), c->d_selftab.as<SelfTab>(), corr,
      sub, panels, c->d_stats.as<unsigned long long>(), curves_dev(c), c->d_mono.as<double>());
  if (has_curves(c)) {
    const int cb = (int)std::min<int64_t>(nblk(n, CURV_WARPS), (int64_t)c->sm_count * 16);
    k_self_curved<P><<<std::max(cb, 1), CURV_WARPS * 32, 0, c->ss>>>(
        n, itgt, ielem, txy, c->d_el.as<ElemRec>(), c->d_coeffs.as<double>(), curves_dev(c), c->d_sx.as<double>(),
        c->d_sy.as<double>(), c->d_sq.as<double>(), c->d_rules.as<RulesDev>(), corr, sub, panels,
        c->d_stats.as<unsigned long long>());
    c->last_launches += 1;
  }
}


// host decode of a sub-simplex path (same child order as decode_path)
static void host_decode_path(unsigned long long path, int d, double v[6]) {
  double ax = 0, ay = 0, bx = 1, by = 0, cx = 0, cy = 1;
  for (int l = d - 1; l >= 0; --l) {
    const int ch = (int)((path >> (2 * l)) & 3ull);
    const double abx = (ax + bx) * 0.5, aby = (ay + by) * 0.5, bcx = (bx + cx) * 0.5, bcy = (by + cy) * 0.5;
    const double cax = (cx + ax) * 0.5, cay = (cy + ay) * 0.5;
    if (ch == 0) { bx = abx; by = aby; cx = cax; cy = cay; }
    else if (ch == 1) { ax = abx; ay = aby; cx = bcx; cy = bcy; }
    else if (ch == 2) { ax = cax; ay = cay; bx = bcx; by = bcy; }
    else { ax = bcx; ay = bcy; bx = cax; by = cay; cx = abx; cy = aby; }
  }
  v[0] = ax; v[1] = ay; v[2] = bx; v[3] = by; v[4] = cx; v[5] = cy;
}

// Build (per evaluation) the per-element near-leaf cache: choose the depth
// D <= cache_max_depth whose cache fits cache_max_bytes, build Vt on the host
// once per (p, rules, D), then contract on the device.
// deepest cached level whose per-element cache fits the byte budget (-1: none)
void decide_cache_depth(vp_ctx* c) {
  if (c->capture) return;  // the eager run's depth
  // default budget: depth 3 for config 4 (1 M elements x 85 slots x 49 nodes
  // = 35 GB) took the deep-leaf kernel 39.6 -> 12.6 ms and the pair stage
  // 222 -> 214 ms against depth 2 within the former 12 GiB
  int64_t budget = c->cache_max_bytes;
  if (budget <= 0) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
      cudaGetLastError();
      free_b = 0;
    }
    budget = std::min<int64_t>(48ll << 30, (int64_t)(free_b / 4) + (int64_t)c->d_gcache.cap);
  }
  int D = std::min(c->cache_max_depth, 6);
  while (D >= 0) {
    const int64_t nslot = ((1ll << (2 * (D + 1))) - 1) / 3;
    if ((double)c->n_tri * nslot * c->rules.len_n * 8.0 <= (double)budget) break;
    --D;
  }
  c->cache_depth = D;
}

int build_near_cache(vp_ctx* c, const int32_t* pelem, int64_t n_pairs) {
  const int Ln = c->rules.len_n, M = c->M;
  const int D = c->cache_depth;
  if (D < 0) return 0;
  // element flags of the call's pairs; only their cache rows are built
  const uint8_t* used = nullptr;
  if (pelem && n_pairs > 0) {
    CUDA_TRY(c, c->d_elused.ensure((size_t)c->n_tri + 1));
    CUDA_TRY(c, cudaMemsetAsync(c->d_elused.p, 0, (size_t)c->n_tri, c->stream));
    k_mark_elems<<<nblk(n_pairs, 256), 256, 0, c->stream>>>(n_pairs, pelem, c->d_elused.as<uint8_t>());
    used = c->d_elused.as<uint8_t>();
    c->last_launches += 1;
  }
  const int64_t nslot = ((1ll << (2 * (D + 1))) - 1) / 3, R = nslot * Ln;
  if (c->cacheV_depth != D || c->cacheV_p != c->p) {
    std::vector<double> Vt((size_t)M * R), kv(M), sref(6 * nslot);
    const vp_rules& r = c->rules;
    for (int d = 0; d <= D; ++d) {
      const int64_t off = ((1ll << (2 * d)) - 1) / 3, n = 1ll << (2 * d);
      for (int64_t path = 0; path < n; ++path) {
        double v[6];
        host_decode_path((unsigned long long)path, d, v);
        double* sr = &sref[6 * (off + path)];
        sr[0] = v[0]; sr[1] = v[1];
        sr[2] = v[2] - v[0]; sr[3] = v[3] - v[1];
        sr[4] = v[4] - v[0]; sr[5] = v[5] - v[1];
        for (int i = 0; i < Ln; ++i) {
          const double u = r.near_x[i], w = r.near_y[i];
          const double xi = v[0] + (u * (v[2] - v[0]) + w * (v[4] - v[0]));
          const double eta = v[1] + (u * (v[3] - v[1]) + w * (v[5] - v[1]));
          koorn_eval(c->p, xi, eta, kv.data());
          const int64_t row = (off + path) * Ln + i;
          // leaf scale 4^-d / (4 pi) folded in; k_near_cache multiplies by det
          const double sc = std::ldexp(1.0, -2 * d) * kInv4Pi;
          for (int j = 0; j < M; ++j) Vt[(size_t)j * R + row] = (r.near_w[i] * kv[j]) * sc;
        }
      }
    }
    CUDA_TRY(c, c->d_cacheV.ensure(sizeof(double) * Vt.size()));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_cacheV.p, Vt.data(), sizeof(double) * Vt.size(), cudaMemcpyHostToDevice,
                                c->stream));
    CUDA_TRY(c, c->d_slotref.ensure(sizeof(double) * sref.size()));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_slotref.p, sref.data(), sizeof(double) * sref.size(), cudaMemcpyHostToDevice,
                                c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->cacheV_depth = D;
    c->cacheV_p = c->p;
  }
  // + one zero row (k_near_cg's rows past a batch point there)
  CUDA_TRY(c, c->d_gcache.ensure(sizeof(double) * (size_t)(c->n_tri * R + Ln + 64)));
  CUDA_TRY(c, cudaMemsetAsync(c->d_gcache.as<double>() + c->n_tri * R, 0, sizeof(double) * (Ln + 64), c->stream));
  static const bool cache_simt = getenv("VP_NEAR_CACHE_SIMT") != nullptr;  // A/B switch: DFMA kernel
  static const bool cache_mma1 = getenv("VP_NEAR_CACHE_MMA1") != nullptr;  // A/B switch: one tile per block
  if (!cache_simt && !cache_mma1) {
    const int64_t nchunk = ((c->n_tri + kNcBM - 1) / kNcBM + kNc2EB - 1) / kNc2EB;
    const int64_t nb = nchunk * nblk(R, kNc2BN);
    if (nb > (int64_t)INT32_MAX) return set_err(c, 1, "near cache: too many blocks");
    k_near_cache_mma2<<<(unsigned)nb, 128, near_cache_mma2_smem(M), c->stream>>>(
        c->n_tri, M, R, c->d_cacheV.as<double>(), c->d_coeffs.as<double>(), c->d_el.as<ElemRec>(),
        c->d_gcache.as<double>(), used);
  } else if (!cache_simt) {
    const int64_t nb = (int64_t)((c->n_tri + kNcBM - 1) / kNcBM) * nblk(R, kNcBN);
    if (nb > (int64_t)INT32_MAX) return set_err(c, 1, "near cache: too many blocks");
    k_near_cache_mma<<<(unsigned)nb, 128, near_cache_mma_smem(M), c->stream>>>(
        c->n_tri, M, R, c->d_cacheV.as<double>(), c->d_coeffs.as<double>(), c->d_el.as<ElemRec>(),
        c->d_gcache.as<double>(), used);
  } else {
    if (nblk(R, 256) > 65535u) return set_err(c, 1, "near cache: too many rows");
    dim3 grid((unsigned)((c->n_tri + kCacheNE - 1) / kCacheNE), (unsigned)nblk(R, 256));
    k_near_cache<<<grid, 256, 0, c->stream>>>(c->n_tri, M, R, c->d_cacheV.as<double>(), c->d_coeffs.as<double>(),
                                              c->d_el.as<ElemRec>(), c->d_gcache.as<double>());
  }
  CUDA_TRY(c, cudaGetLastError());
  c->last_launches += 1;
  return 0;
}

// Sample set and map of the self kernel's density step (SelfTab::T2).
// Points: approximate Fekete points of degree p on the reference triangle,
// chosen by column-pivoted Gram-Schmidt on the orthonormal Koornwinder
// basis over a 60 x 60 lattice (ties -> lowest index); Lebesgue constant
// 2.7 / 4.8 / 11.2 / 17.3 at p = 4 / 6 / 8 / 12 (the shifted lattice of the
// targets: 129 / 769 / 4097 / 98305).  (xi, eta) -> (r, s) = (1 - xi, eta).
// T2 = Tgrid . R, where R [(p+1)^2 x M] interpolates the Gauss-Legendre grid
// (r_a, r_a sigma_b) from the samples and Tgrid [2(p+1) x (p+1)^2] is the
// PL / PM / moment chain of k_self; long double throughout.
int self_sample_map(vp_ctx* c, SelfTab& T, const double* gx_m11) {
  const int p = c->p, np = p + 1, M = koorn_size(p);
  constexpr int G = 60;
  std::vector<double> cx, cy;
  for (int j = 0; j <= G; ++j)
    for (int i = 0; i + j <= G; ++i) {
      cx.push_back((double)i / G);
      cy.push_back((double)j / G);
    }
  const int nc = (int)cx.size();
  std::vector<long double> A((size_t)nc * M);
  std::vector<double> kv(M);
  for (int q = 0; q < nc; ++q) {
    koorn_eval(p, cx[q], cy[q], kv.data());
    for (int i = 0; i < M; ++i) A[(size_t)q * M + i] = kv[i];
  }
  std::vector<long double> nrm(nc);
  std::vector<char> used(nc, 0);
  std::vector<int> sel;
  for (int q = 0; q < nc; ++q) {
    long double v = 0.0L;
    for (int i = 0; i < M; ++i) v += A[(size_t)q * M + i] * A[(size_t)q * M + i];
    nrm[q] = v;
  }
  for (int k = 0; k < M; ++k) {
    int best = -1;
    for (int q = 0; q < nc; ++q)
      if (!used[q] && (best < 0 || nrm[q] > nrm[best])) best = q;
    if (best < 0 || !(nrm[best] > 0.0L)) return set_err(c, 2, "self table: sample selection failed");
    used[best] = 1;
    sel.push_back(best);
    const long double inv = 1.0L / std::sqrt(nrm[best]);
    std::vector<long double> qv(M);
    for (int i = 0; i < M; ++i) qv[i] = A[(size_t)best * M + i] * inv;
    for (int q = 0; q < nc; ++q) {
      if (used[q]) continue;
      long double d = 0.0L;
      for (int i = 0; i < M; ++i) d += qv[i] * A[(size_t)q * M + i];
      long double v = 0.0L;
      for (int i = 0; i < M; ++i) {
        A[(size_t)q * M + i] -= d * qv[i];
        v += A[(size_t)q * M + i] * A[(size_t)q * M + i];
      }
      nrm[q] = v;
    }
  }
  // B [M x M] = K_i at the samples (rows = samples); Binv by Gauss-Jordan
  std::vector<long double> B((size_t)M * M), Bi((size_t)M * M, 0.0L);
  for (int q = 0; q < M; ++q) {
    koorn_eval(p, cx[sel[q]], cy[sel[q]], kv.data());
    for (int i = 0; i < M; ++i) B[(size_t)q * M + i] = kv[i];
    Bi[(size_t)q * M + q] = 1.0L;
    T.sr[q] = 1.0 - cx[sel[q]];
    T.ss[q] = cy[sel[q]];
  }
  for (int col = 0; col < M; ++col) {
    int piv = col;
    for (int r = col + 1; r < M; ++r)
      if (std::fabs(B[(size_t)r * M + col]) > std::fabs(B[(size_t)piv * M + col])) piv = r;
    if (!(std::fabs(B[(size_t)piv * M + col]) > 0.0L)) return set_err(c, 2, "self table: singular sample matrix");
    for (int k = 0; k < M; ++k) {
      std::swap(B[(size_t)col * M + k], B[(size_t)piv * M + k]);
      std::swap(Bi[(size_t)col * M + k], Bi[(size_t)piv * M + k]);
    }
    const long double d = 1.0L / B[(size_t)col * M + col];
    for (int k = 0; k < M; ++k) {
      B[(size_t)col * M + k] *= d;
      Bi[(size_t)col * M + k] *= d;
    }
    for (int r = 0; r < M; ++r) {
      if (r == col) continue;
      const long double f = B[(size_t)r * M + col];
      if (f == 0.0L) continue;
      for (int k = 0; k < M; ++k) {
        B[(size_t)r * M + k] -= f * B[(size_t)col * M + k];
        Bi[(size_t)r * M + k] -= f * Bi[(size_t)col * M + k];
      }
    }
  }
  // (B^-1 maps sample values to Koornwinder coefficients: coef = Binv f since
  // f_q = sum_i B[q][i] coef_i.)  R[(a,b)][q] = sum_i K_i(grid ab) Binv[i][q].
  const bool horner = p <= kSelfHornerMaxP;
  std::vector<long double> Tg((size_t)2 * np * np * np, 0.0L);  // [o][(a,b)]
  for (int kk = 0; kk < np; ++kk)
    for (int a = 0; a < np; ++a)
      for (int b = 0; b < np; ++b) {
        const long double pm = horner ? T.PM[kk * np + b] : T.PL[kk * np + b];
        long double sb = 0.0L, sc = 0.0L;
        for (int n = 0; n < np; ++n) {
          sb += (long double)T.bt[n] * T.PL[n * np + a];
          sc += (long double)T.ct[n] * T.PL[n * np + a];
        }
        Tg[(size_t)kk * np * np + a * np + b] = sb * pm;
        Tg[(size_t)(np + kk) * np * np + a * np + b] = sc * pm;
      }
  std::vector<long double> T2((size_t)2 * np * M, 0.0L);
  for (int a = 0; a < np; ++a)
    for (int b = 0; b < np; ++b) {
      const double r = 0.5 * (gx_m11[a] + 1.0), sg = 0.5 * (gx_m11[b] + 1.0);
      koorn_eval(p, 1.0 - r, r * sg, kv.data());
      for (int q = 0; q < M; ++q) {
        long double rq = 0.0L;
        for (int i = 0; i < M; ++i) rq += (long double)kv[i] * Bi[(size_t)i * M + q];
        for (int o = 0; o < 2 * np; ++o) T2[(size_t)o * M + q] += Tg[(size_t)o * np * np + a * np + b] * rq;
      }
    }
  for (size_t i = 0; i < T2.size(); ++i) T.T2[i] = (double)T2[i];
  return 0;
}

// Kmon [M x M]: row j = the monomial coefficients of c_j K_j (the normalised
// Koornwinder basis of koorn.cuh / koornwinder.hpp:12-21) in (X, Y) =
// (xi - c0, eta - c0), c0 = kMonoC0, column mono_off(p, j') + i' for
// X^i' Y^j'.  Built by the basis recurrences of koorn_eval carried out on
// bivariate polynomials in long double, so each entry is the exact
// coefficient up to long-double rounding.
static void mono_table(int p, std::vector<double>& out) {
  const int n = p + 1, M = koorn_size(p);
  using Poly = std::vector<long double>;  // [i * n + j] = coefficient of X^i Y^j, i + j <= p
  auto zero = [&] { return Poly((size_t)n * n, 0.0L); };
  auto mul = [&](const Poly& a, const Poly& b) {
    Poly r = zero();
    for (int i = 0; i < n; ++i)
      for (int j = 0; i + j < n; ++j) {
        const long double av = a[(size_t)i * n + j];
        if (av == 0.0L) continue;
        for (int k = 0; i + k < n; ++k)
          for (int l = 0; i + j + k + l < n; ++l) r[(size_t)(i + k) * n + j + l] += av * b[(size_t)k * n + l];
      }
    return r;
  };
  auto lin = [&](long double a, const Poly& x, long double b, const Poly& y) {
    Poly r = zero();
    for (size_t i = 0; i < r.size(); ++i) r[i] = a * x[i] + b * y[i];
    return r;
  };
  const long double c0 = (long double)kMonoC0;
  Poly one = zero(), x = zero(), y = zero();
  one[0] = 1.0L;
  x[0] = c0;
  y[0] = c0;
  if (p >= 1) {
    x[(size_t)1 * n] = 1.0L;
    y[1] = 1.0L;
  }
  const Poly v = lin(1.0L, one, -1.0L, x);  // 1 - x
  const Poly u = lin(2.0L, y, -1.0L, v);    // 2y - (1 - x)
  const Poly v2 = mul(v, v);
  const Poly t = lin(2.0L, x, -1.0L, one);  // 2x - 1
  std::vector<Poly> L{one};
  if (p >= 1) L.push_back(u);
  for (int m = 1; m + 1 <= p; ++m)
    L.push_back(lin((long double)(2 * m + 1) / (m + 1), mul(u, L[m]), -(long double)m / (m + 1), mul(v2, L[m - 1])));
  out.assign((size_t)M * M, 0.0);
  for (int m = 0; m <= p; ++m) {
    const long double a = 2 * m + 1;
    std::vector<Poly> P{one};
    if (m + 1 <= p) P.push_back(lin(0.5L * (a + 2.0L), t, 0.5L * a, one));
    for (int k = 1; m + k + 1 <= p; ++k) {
      const long double kk = k;
      const long double c1 = 2 * (kk + 1) * (kk + a + 1) * (2 * kk + a);
      const long double c2 = (2 * kk + a + 1) * (a * a);
      const long double c3 = (2 * kk + a) * (2 * kk + a + 1) * (2 * kk + a + 2);
      const long double c4 = 2 * (kk + a) * kk * (2 * kk + a + 2);
      Poly nx = lin(c2 / c1, P[k], c3 / c1, mul(t, P[k]));
      P.push_back(lin(1.0L, nx, -c4 / c1, P[k - 1]));
    }
    for (int k = 0; m + k <= p; ++k) {
      const int nn = m + k, row = koorn_index(m, nn);
      const long double cn = std::sqrt((long double)((2 * m + 1) * (2 * nn + 2)));
      const Poly b = mul(P[k], L[m]);
      for (int i = 0; i < n; ++i)
        for (int j = 0; i + j < n; ++j) out[(size_t)row * M + mono_off(p, j) + i] = (double)(cn * b[(size_t)i * n + j]);
    }
  }
}

// SelfTab for the current (p, GGQ rule): Gauss-Legendre interpolation grid
// on [0,1], Legendre projection weights and the GGQ-rule moments.
int upload_self_tab(vp_ctx* c) {
  if (!c->have_rules || c->p < 0) return 0;
  SelfTab T;
  std::memset(&T, 0, sizeof(T));
  const int np = c->p + 1;
  T.np = np;
  double gx[kMaxPdev + 1], gw[kMaxPdev + 1];
  if (vps_gauss_legendre(np, gx, gw) != 0) return set_err(c, 1, "self table: Gauss-Legendre failed");
  auto legendre = [](int n, double x) {
    double p0 = 1.0, p1 = x;
    if (n == 0) return 1.0;
    for (int k = 1; k < n; ++k) {
      const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
      p0 = p1;
      p1 = p2;
    }
    return p1;
  };
  for (int a = 0; a < np; ++a) T.gx[a] = 0.5 * (gx[a] + 1.0);
  for (int n = 0; n < np; ++n)
    for (int a = 0; a < np; ++a) T.PL[n * np + a] = (2 * n + 1) * (0.5 * gw[a]) * legendre(n, gx[a]);
  const vp_rules& r = c->rules;
  for (int n = 0; n < np; ++n) {
    double b = 0.0, cc = 0.0;
    for (int j = 0; j <= r.n_g; ++j) {
      const double rj = r.ggq_r[j], wj = r.ggq_w[j], pn = legendre(n, 2.0 * rj - 1.0);
      b += wj * rj * pn;
      cc += wj * rj * std::log(rj) * pn;
    }
    T.bt[n] = b;
    T.ct[n] = cc;
    T.la[n] = double(2 * n + 1) / double(n + 1);
    T.lb[n] = double(n) / double(n + 1);
  }
  {
    // monomial coefficients of P_k: mc[k][j] = [x^j] P_k(x), long double recurrence
    std::vector<long double> mc((size_t)np * np, 0.0L);
    mc[0] = 1.0L;
    if (np > 1) mc[1 * np + 1] = 1.0L;
    for (int k = 1; k + 1 < np; ++k)
      for (int j = 0; j < np; ++j) {
        long double v = -(long double)k * mc[(size_t)(k - 1) * np + j];
        if (j > 0) v += (long double)(2 * k + 1) * mc[(size_t)k * np + j - 1];
        mc[(size_t)(k + 1) * np + j] = v / (long double)(k + 1);
      }
    for (int j = 0; j < np; ++j)
      for (int a = 0; a < np; ++a) {
        long double v = 0.0L;
        for (int k = 0; k < np; ++k)
          v += mc[(size_t)k * np + j] * (long double)(2 * k + 1) * (0.5L * gw[a]) * (long double)legendre(k, gx[a]);
        T.PM[j * np + a] = (double)v;
      }
  }
  if (int rc = self_sample_map(c, T, gx)) return rc;
  if (c->p <= kMonoMaxP) {
    std::vector<double> km;
    mono_table(c->p, km);
    CUDA_TRY(c, c->d_kmon.ensure(sizeof(double) * km.size()));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_kmon.p, km.data(), sizeof(double) * km.size(), cudaMemcpyHostToDevice, c->stream));
  }
  CUDA_TRY(c, c->d_selftab.ensure(sizeof(SelfTab)));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_selftab.p, &T, sizeof(SelfTab), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->selftab_p = c->p;
  return 0;
}

int ensure_ready(vp_ctx* c, bool need_density) {
  if (!c) return 1;
  if (!c->have_mesh) return set_err(c, 1, "usage: vp_set_mesh must precede evaluation");
  if (!c->have_rules) return set_err(c, 1, "usage: vp_set_rules must precede evaluation");
  if (need_density && !c->have_density) return set_err(c, 1, "usage: vp_set_density must precede evaluation");
  if (!c->elems_ok)
    return set_err(c, 1, "usage: the mesh and rules were rejected by vp_set_mesh/vp_set_rules (see that error)");
  return 0;
}

int compute_sources(vp_ctx* c) {
  if (c->sources_valid) return 0;
  const int64_t S = c->n_tri * c->rules.len_q;
  CUDA_TRY(c, c->d_sx.ensure(sizeof(double) * S));
  CUDA_TRY(c, c->d_sy.ensure(sizeof(double) * S));
  CUDA_TRY(c, c->d_sq.ensure(sizeof(double) * S));
  k_sources<<<nblk(S, 256), 256, 0, c->stream>>>(c->n_tri, c->rules.len_q, c->M, c->d_el.as<ElemRec>(),
                                                  c->d_coeffs.as<double>(), c->d_V.as<double>(),
                                                  c->d_rules.as<RulesDev>(), c->d_sx.as<double>(),
                                                  c->d_sy.as<double>(), c->d_sq.as<double>());
  if (c->p <= kMonoMaxP) {  // K5's density samples
    const int64_t n = c->n_tri * c->M;
    CUDA_TRY(c, c->d_mono.ensure(sizeof(double) * n));
    k_mono<<<nblk(n, 256), 256, 0, c->stream>>>(c->n_tri, c->M, c->d_coeffs.as<double>(), c->d_kmon.as<double>(),
                                                c->d_mono.as<double>());
    c->last_launches += 1;
  }
  if (has_curves(c)) {
    const int64_t nc = (int64_t)c->h_celist.size();
    k_sources_curved<<<nblk(nc * c->rules.len_q, 128), 128, 0, c->stream>>>(
        nc, c->d_celist.as<int32_t>(), c->rules.len_q, c->d_el.as<ElemRec>(), curves_dev(c),
        c->d_rules.as<RulesDev>(), c->d_sx.as<double>(), c->d_sy.as<double>(), c->d_sq.as<double>());
    c->last_launches += 1;
  }
  CUDA_TRY(c, cudaGetLastError());
  c->sources_valid = true;
  c->last_launches += 1;
  return 0;
}

constexpr size_t kFarSmem = sizeof(double2) * kFarLogEntries * kFarCopies + FAR_TILE * (sizeof(double2) + sizeof(double));

int direct_far_sum(vp_ctx* c, int64_t T, const double2* txy, double* ufar, bool zero_check, DevBuf& part);
int fmm_far_sum(vp_ctx* c, int64_t T, const double2* txy, double* ufar, bool zero_check);

// the far field on stream c->fs (c->stream unless the caller overlaps it);
// its launches are counted in c->far_launches
int far_sum(vp_ctx* c, int64_t T, const double2* txy, double* ufar, bool zero_check) {
  if (c->far_method == 1) return fmm_far_sum(c, T, txy, ufar, zero_check);
  return direct_far_sum(c, T, txy, ufar, zero_check, c->d_part);
}

int direct_far_sum(vp_ctx* c, int64_t T, const double2* txy, double* ufar, bool zero_check, DevBuf& part) {
  const int64_t S = c->n_tri * c->rules.len_q;
  // The source chunking depends on S only, never on T: every target's far
  // sum is the same fixed-order sum of chunk partials however the targets
  // are batched or sharded (bitwise shard invariance).  Up to 256 chunks of
  // >= 4096 sources: enough (target block, chunk) blocks that the last wave
  // of one-block-per-SM launches is a small fraction (config 4 subset: 28 x
  // 256 blocks = 48.4 waves of 148, against 12.1 waves with 64 chunks).
  int64_t chunk = std::max<int64_t>(4096, (S + 255) / 256);
  chunk = (chunk + FAR_TILE - 1) / FAR_TILE * FAR_TILE;
  const int nsplit = (int)std::max<int64_t>(1, (S + chunk - 1) / chunk);
  // Targets per thread: 8 (the fastest per pair), or 4 when a target count
  // that is not a multiple of 4,096 would leave the last block of 8-target
  // threads mostly idle (one block per SM, so a block is the unit of time):
  // the cost model is waves x targets per block x per-pair speed (4-target
  // threads measured ~3 % slower per pair).  A strong-scaled shard of the
  // config-4 subset at 8 GPUs (14,336 targets = 3.5 x 4,096) takes 4.  Each
  // target's sum is the same fixed-order sum either way (bitwise invariant).
  auto cost = [&](int r) {
    const int64_t tb = (int64_t)FAR_THREADS * r;
    const double waves = std::ceil((double)nblk(T, (int)tb) * nsplit / (double)c->sm_count);
    return waves * (double)tb * (r == 4 ? 1.03 : 1.0);
  };
  static const int forced = std::getenv("VP_FAR_TPT") ? std::atoi(std::getenv("VP_FAR_TPT")) : 0;  // A/B: 4 or 8
  const int R = forced == 4 || forced == 8 ? (forced == 4 ? 4 : FAR_R) : (FAR_R == 8 && cost(4) < cost(8)) ? 4 : FAR_R;
  // targets in batches so the [nsplit x batch] partials stay within 1 GiB
  const int64_t tblk = (int64_t)FAR_THREADS * R;
  const int64_t batch = std::max<int64_t>(tblk, ((1ll << 27) / nsplit) / tblk * tblk);
  const int64_t Tb = std::min<int64_t>(T, batch);
  CUDA_TRY(c, part.ensure(sizeof(double) * std::max<int64_t>(Tb, 1) * nsplit));
  for (int64_t t0 = 0; t0 < T; t0 += batch) {
    const int64_t n = std::min<int64_t>(batch, T - t0);
    dim3 grid((unsigned)nblk(n, (int)tblk), (unsigned)nsplit);
    auto kern = zero_check ? (R == 4 ? k_far<true, 4> : k_far<true, FAR_R>) : (R == 4 ? k_far<false, 4> : k_far<false, FAR_R>);
    kern<<<grid, FAR_THREADS, kFarSmem, c->fs>>>(n, txy + t0, S, c->d_sx.as<double>(), c->d_sy.as<double>(),
                                                 c->d_sq.as<double>(), chunk, part.as<double>(), 0x3ff00000u);
    k_far_reduce<<<nblk(n, 256), 256, 0, c->fs>>>(n, nsplit, part.as<double>(), ufar + t0);
    c->far_launches += 2;
  }
  CUDA_TRY(c, cudaGetLastError());
  return 0;
}

// FMM far field (vp_fmm.cuh).  The tree is built from the sources only
// (root = mesh bbox + margin), so u(t) does not depend on the target set.
int fmm_far_sum(vp_ctx* c, int64_t T, const double2* txy, double* ufar, bool zero_check) {
  const int64_t S = c->n_tri * c->rules.len_q;
  const int p = c->fmm_p, P1 = p + 1;
  FmmGeom g;
  const double W = c->bx1 - c->bx0, H = c->by1 - c->by0;
  g.h0 = std::max(W, H) * (1.0 + 1.0 / 64.0);
  if (!(g.h0 > 0.0)) g.h0 = 1.0;
  g.x0 = 0.5 * (c->bx0 + c->bx1) - 0.5 * g.h0;
  g.y0 = 0.5 * (c->by0 + c->by1) - 0.5 * g.h0;
  g.p = p;
  int L = (int)std::lround(0.5 * std::log2(std::max(1.0, (double)S / std::max(1, c->fmm_leaf))));
  g.L = L = std::max(2, std::min(11, L));
  c->fmm_levels = L;
  const int64_t nleaf = 1ll << (2 * L);
  const int64_t nbox = ((1ll << (2 * (L + 1))) - 1) / 3;
  FmmTabLayout TL(p);
  if (c->tab_p != p) {
    std::vector<double> tab;
    fmm_tables_fill(p, tab);
    CUDA_TRY(c, c->f_tab.ensure(sizeof(double) * tab.size()));
    CUDA_TRY(c, cudaMemcpyAsync(c->f_tab.p, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice,
                                c->fs));
    CUDA_TRY(c, cudaStreamSynchronize(c->fs));
    c->tab_p = p;
  }
  // bin and sort the sources by leaf box (stable: source order kept within a box)
  CUDA_TRY(c, c->f_keys.ensure(sizeof(int32_t) * S));
  CUDA_TRY(c, c->f_keys2.ensure(sizeof(int32_t) * S));
  CUDA_TRY(c, c->f_vals.ensure(sizeof(int32_t) * S));
  CUDA_TRY(c, c->f_idx.ensure(sizeof(int32_t) * S));
  CUDA_TRY(c, c->f_beg.ensure(sizeof(int64_t) * nleaf));
  CUDA_TRY(c, c->f_end.ensure(sizeof(int64_t) * nleaf));
  CUDA_TRY(c, c->f_pxy.ensure(sizeof(double2) * S));
  CUDA_TRY(c, c->f_pq.ensure(sizeof(double) * S));
  CUDA_TRY(c, c->f_mp.ensure(sizeof(double2) * nbox * P1));
  CUDA_TRY(c, c->f_lp.ensure(sizeof(double2) * nbox * P1));
  k_fmm_keys<<<nblk(S, 256), 256, 0, c->fs>>>(S, c->d_sx.as<double>(), c->d_sy.as<double>(), g,
                                                   c->f_keys.as<int32_t>(), c->f_vals.as<int32_t>());
  size_t tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, c->f_keys.as<int32_t>(), c->f_keys2.as<int32_t>(),
                                  c->f_vals.as<int32_t>(), c->f_idx.as<int32_t>(), (int)S, 0, 2 * L, c->fs);
  CUDA_TRY(c, c->f_tmp.ensure(tmpb));
  cub::DeviceRadixSort::SortPairs(c->f_tmp.p, tmpb, c->f_keys.as<int32_t>(), c->f_keys2.as<int32_t>(),
                                  c->f_vals.as<int32_t>(), c->f_idx.as<int32_t>(), (int)S, 0, 2 * L, c->fs);
  CUDA_TRY(c, cudaMemsetAsync(c->f_beg.p, 0, sizeof(int64_t) * nleaf, c->fs));
  CUDA_TRY(c, cudaMemsetAsync(c->f_end.p, 0, sizeof(int64_t) * nleaf, c->fs));
  k_cell_ranges<<<nblk(S, 256), 256, 0, c->fs>>>(S, c->f_keys2.as<int32_t>(), c->f_beg.as<int64_t>(),
                                                      c->f_end.as<int64_t>());
  k_fmm_gather<<<nblk(S, 256), 256, 0, c->fs>>>(S, c->f_idx.as<int32_t>(), c->d_sx.as<double>(),
                                                     c->d_sy.as<double>(), c->d_sq.as<double>(),
                                                     c->f_pxy.as<double2>(), c->f_pq.as<double>());
  // targets in leaf order (stable radix sort by leaf key) and the boxes that hold them
  CUDA_TRY(c, c->f_flag.ensure(sizeof(int32_t) * (T + 1)));
  CUDA_TRY(c, c->f_tk.ensure(sizeof(int32_t) * (T + 1)));
  CUDA_TRY(c, c->f_tk2.ensure(sizeof(int32_t) * (T + 1)));
  CUDA_TRY(c, c->f_tv.ensure(sizeof(int32_t) * (T + 1)));
  CUDA_TRY(c, c->f_tord.ensure(sizeof(int32_t) * (T + 1)));
  k_fmm_tkeys<<<nblk(T, 256), 256, 0, c->fs>>>(T, txy, g, c->f_tk.as<int32_t>(), c->f_tv.as<int32_t>());
  tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, c->f_tk.as<int32_t>(), c->f_tk2.as<int32_t>(), c->f_tv.as<int32_t>(),
                                  c->f_tord.as<int32_t>(), (int)T, 0, 2 * L + 1, c->fs);
  CUDA_TRY(c, c->f_tmp.ensure(tmpb));
  cub::DeviceRadixSort::SortPairs(c->f_tmp.p, tmpb, c->f_tk.as<int32_t>(), c->f_tk2.as<int32_t>(),
                                  c->f_tv.as<int32_t>(), c->f_tord.as<int32_t>(), (int)T, 0, 2 * L + 1, c->fs);
  CUDA_TRY(c, c->f_active.ensure((size_t)nbox));
  static const bool all_boxes = getenv("VP_FMM_ALL_BOXES") != nullptr;  // A/B switch: no skipping
  CUDA_TRY(c, cudaMemsetAsync(c->f_active.p, all_boxes ? 1 : 0, (size_t)nbox, c->fs));
  k_fmm_mark_leaves<<<nblk(T, 256), 256, 0, c->fs>>>(T, c->f_tk.as<int32_t>(), L, c->f_active.as<uint8_t>());
  for (int l = L - 1; l >= 2; --l)
    k_fmm_mark_parents<<<nblk(1ll << (2 * l), 256), 256, 0, c->fs>>>(l, c->f_active.as<uint8_t>());
  // upward pass
  const int wblocks = (int)std::min<int64_t>(nblk(nleaf, kFmmThreads / 32), (int64_t)c->sm_count * 64);
  const size_t sm_p2m = sizeof(double2) * (kFmmThreads / 32) * 32 * (size_t)(P1 | 1);
  k_fmm_p2m<<<std::max(wblocks, 1), kFmmThreads, sm_p2m, c->fs>>>(g, c->f_beg.as<int64_t>(), c->f_end.as<int64_t>(),
                                                                  c->f_pxy.as<double2>(), c->f_pq.as<double>(),
                                                                  c->f_mp.as<double2>());
  const size_t P1e = ((size_t)P1 * P1 + 1) & ~(size_t)1;
  const size_t sm_m2m = sizeof(double) * (P1e + 8 * P1);
  for (int l = L - 1; l >= 2; --l) {
    const int64_t nb = 1ll << (2 * l);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(nblk(nb, kFmmThreads / 32), (int64_t)c->sm_count * 64));
    k_fmm_m2m<<<blocks, kFmmThreads, sm_m2m, c->fs>>>(g, l, c->f_tab.as<double>(), c->f_mp.as<double2>());
  }
  // downward pass
  const size_t sm_m2l = sizeof(double) * (2 * P1e + 8 * P1 + 2 * (kFmmThreads / 32) * P1);
  for (int l = 2; l <= L; ++l) {
    const int64_t nb = 1ll << (2 * l);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(nblk(nb, kFmmThreads / 32), (int64_t)c->sm_count * 64));
#define VP_M2L_CASE(N)                                                                                   \
  case N:                                                                                                \
    k_fmm_m2l32<N><<<blocks, kFmmThreads, 0, c->fs>>>(g, l, c->f_tab.as<double>(), c->f_mp.as<double2>(), \
                                                      c->f_lp.as<double2>(), c->f_active.as<uint8_t>()); \
    break;
    switch (P1) {  // one coefficient per lane for the orders of vp_fmm_order_for
      VP_M2L_CASE(8) VP_M2L_CASE(12) VP_M2L_CASE(16) VP_M2L_CASE(20) VP_M2L_CASE(24) VP_M2L_CASE(28) VP_M2L_CASE(32)
      default:
        k_fmm_m2l<<<blocks, kFmmThreads, sm_m2l, c->fs>>>(g, l, c->f_tab.as<double>(), c->f_mp.as<double2>(),
                                                          c->f_lp.as<double2>(), c->f_active.as<uint8_t>());
    }
#undef VP_M2L_CASE
  }
  // L2P + P2P over the targets in leaf order
  const size_t sm_eval = sizeof(LogTab);
  if (zero_check)
    k_fmm_eval<true><<<nblk(T, 256), 256, sm_eval, c->fs>>>(
        T, txy, g, c->f_beg.as<int64_t>(), c->f_end.as<int64_t>(), c->f_pxy.as<double2>(), c->f_pq.as<double>(),
        c->f_lp.as<double2>(), ufar, c->f_flag.as<int32_t>(), 0x3ff00000u, c->f_tord.as<int32_t>());
  else
    k_fmm_eval<false><<<nblk(T, 256), 256, sm_eval, c->fs>>>(
        T, txy, g, c->f_beg.as<int64_t>(), c->f_end.as<int64_t>(), c->f_pxy.as<double2>(), c->f_pq.as<double>(),
        c->f_lp.as<double2>(), ufar, c->f_flag.as<int32_t>(), 0x3ff00000u, c->f_tord.as<int32_t>());
  c->far_launches += 3;
  CUDA_TRY(c, cudaGetLastError());
  c->far_launches += 8 + 3 * (L - 1) - 1;
  // targets outside the root box: direct far sum
  CUDA_TRY(c, c->f_oidx.ensure(sizeof(int32_t) * (T + 1)));
  CUDA_TRY(c, c->f_cnt.ensure(sizeof(int64_t)));
  tmpb = 0;
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tmpb, it, c->f_flag.as<int32_t>(), c->f_oidx.as<int32_t>(),
                             c->f_cnt.as<int64_t>(), (int)T, c->fs);
  CUDA_TRY(c, c->f_tmp.ensure(tmpb));
  cub::DeviceSelect::Flagged(c->f_tmp.p, tmpb, it, c->f_flag.as<int32_t>(), c->f_oidx.as<int32_t>(),
                             c->f_cnt.as<int64_t>(), (int)T, c->fs);
  int64_t nout = 0;
  if (c->capture) {
    nout = c->plan.fmm_nout;
  } else {
    CUDA_TRY(c, cudaMemcpyAsync(&nout, c->f_cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, c->fs));
    CUDA_TRY(c, cudaStreamSynchronize(c->fs));
    c->plan.fmm_nout = nout;
  }
  c->fmm_outside = nout;
  if (nout > 0) {
    CUDA_TRY(c, c->f_otxy.ensure(sizeof(double2) * nout));
    CUDA_TRY(c, c->f_ou.ensure(sizeof(double) * nout));
    k_gather_targets<<<nblk(nout, 256), 256, 0, c->fs>>>(nout, c->f_oidx.as<int32_t>(), txy,
                                                              c->f_otxy.as<double2>());
    if (int rc = direct_far_sum(c, nout, c->f_otxy.as<double2>(), c->f_ou.as<double>(), zero_check, c->d_part))
      return rc;
    k_scatter_add<<<nblk(nout, 256), 256, 0, c->fs>>>(nout, c->f_oidx.as<int32_t>(), c->f_ou.as<double>(), ufar);
    c->far_launches += 2;
  }
  return 0;
}

// list build into ctx buffers: self, cnt, off (T+1), ids, selfref
int build_lists(vp_ctx* c, int64_t T, const double2* txy, int64_t* n_ids_out) {
  CUDA_TRY(c, c->d_self.ensure(sizeof(int32_t) * (T + 1)));
  CUDA_TRY(c, c->d_cnt.ensure(sizeof(int64_t) * (T + 1)));
  CUDA_TRY(c, c->d_off.ensure(sizeof(int64_t) * (T + 1)));
  CUDA_TRY(c, c->d_selfref.ensure(sizeof(double2) * (T + 1)));
  const int cap = 16;  // N(t) ids kept by the count pass (|N(t)| ~ 1-7 on the configs)
  CUDA_TRY(c, c->d_lsc.ensure(sizeof(int32_t) * (size_t)T * cap + 4));
  CUDA_TRY(c, c->d_tover.ensure(sizeof(int32_t) * (T + 1)));
  CUDA_TRY(c, c->d_ntover.ensure(sizeof(unsigned)));
  CUDA_TRY(c, c->d_err.ensure(2 * sizeof(int)));  // [0] near-field limits, [1] non-finite target
  CUDA_TRY(c, cudaMemsetAsync(c->d_ntover.p, 0, sizeof(unsigned), c->stream));
  const GridDev G = c->grid;
  const int nan = (int)c->h_allnear.size();
  (has_curves(c) ? k_lists<false, true> : k_lists<false, false>)<<<nblk(T, 128), 128, 0, c->stream>>>(
      T, txy, c->d_el.as<ElemRec>(), c->d_bbf.as<float4>(), G, c->d_cbeg.as<int64_t>(), c->d_cend.as<int64_t>(),
      c->d_celems.as<int32_t>(), c->d_allnear.as<int32_t>(), nan, c->d_self.as<int32_t>(),
      c->d_cnt.as<int64_t>(), nullptr, nullptr, c->d_selfref.as<double2>(), curves_dev(c), nullptr,
      c->d_lsc.as<int32_t>(), cap, c->d_tover.as<int32_t>(), c->d_ntover.as<unsigned>(), c->d_err.as<int>() + 1);
  CUDA_TRY(c, cudaMemsetAsync(c->d_cnt.as<int64_t>() + T, 0, sizeof(int64_t), c->stream));
  size_t tmpb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmpb, c->d_cnt.as<int64_t>(), c->d_off.as<int64_t>(), T + 1, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceScan::ExclusiveSum(c->d_tmp.p, tmpb, c->d_cnt.as<int64_t>(), c->d_off.as<int64_t>(), T + 1, c->stream);
  int64_t n_ids = 0;
  unsigned nover = 0;
  if (c->capture) {
    n_ids = c->plan.n_ids;
    nover = c->plan.list_nover;
  } else {
    CUDA_TRY(c, cudaMemcpyAsync(&n_ids, c->d_off.as<int64_t>() + T, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(&nover, c->d_ntover.p, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->plan.n_ids = n_ids;
    c->plan.list_nover = nover;
  }
  CUDA_TRY(c, c->d_ids.ensure(sizeof(int32_t) * (n_ids + 1)));
  k_lists_copy<<<nblk(T, 256), 256, 0, c->stream>>>(T, c->d_off.as<int64_t>(), cap, c->d_lsc.as<int32_t>(),
                                                    c->d_ids.as<int32_t>());
  if (nover > 0)
    (has_curves(c) ? k_lists<true, true> : k_lists<true, false>)<<<nblk(nover, 128), 128, 0, c->stream>>>(
        nover, txy, c->d_el.as<ElemRec>(), c->d_bbf.as<float4>(), G, c->d_cbeg.as<int64_t>(),
        c->d_cend.as<int64_t>(),
        c->d_celems.as<int32_t>(), c->d_allnear.as<int32_t>(), nan, nullptr, nullptr, c->d_off.as<int64_t>(),
        c->d_ids.as<int32_t>(), nullptr, curves_dev(c), c->d_tover.as<int32_t>(), nullptr, 0, nullptr, nullptr,
        nullptr);
  CUDA_TRY(c, cudaGetLastError());
  c->last_launches += 3 + (nover > 0 ? 1 : 0);
  *n_ids_out = n_ids;
  return 0;
}

int evaluate_impl(vp_ctx* c, int64_t T, const double2* txy, double* u, vp_stats* st) {
  c->last_launches = 0;
  CUDA_TRY(c, c->d_stats.ensure(sizeof(unsigned long long) * 8));
  CUDA_TRY(c, c->d_err.ensure(2 * sizeof(int)));
  CUDA_TRY(c, cudaMemsetAsync(c->d_stats.p, 0, sizeof(unsigned long long) * 8, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->d_err.p, 0, 2 * sizeof(int), c->stream));
  cudaEvent_t* ev = c->ev;
  CUDA_TRY(c, cudaEventRecord(ev[0], c->stream));
  int64_t n_ids = 0;
  if (int rc = build_lists(c, T, txy, &n_ids)) return rc;
  CUDA_TRY(c, cudaEventRecord(ev[1], c->stream));
  c->sources_valid = false;  // strengths are part of every evaluation pass
  if (int rc = compute_sources(c)) return rc;
  CUDA_TRY(c, cudaEventRecord(ev[6], c->stream));
  CUDA_TRY(c, c->d_ufar.ensure(sizeof(double) * (T + 1)));
  c->far_launches = 0;
  // FMM: the far field overlaps the near and self stages, on its own stream
  // and host thread (its host syncs then wait on that stream only).  The
  // direct K2 fills every SM by itself, so it runs alone and its per-kernel
  // timing stays clean.
  const bool overlap = c->far_method == 1;
  int far_rc = 0;
  // on an error return after s2/s3 were forked, wait for their work (it reads
  // the caller's targets and updates d_stats) before the next call reuses the
  // buffers; declared first, so it runs after FarJoin joined the far thread
  struct ForkGuard {
    vp_ctx* c;
    bool ok = false;
    ~ForkGuard() {
      if (!ok) {
        cudaStreamSynchronize(c->s3);
        cudaStreamSynchronize(c->s2);
      }
    }
  } fork_guard{c};
  std::thread far_thread;
  struct FarJoin {  // joins on every return path and restores the far stream
    vp_ctx* c;
    std::thread& t;
    ~FarJoin() {
      if (t.joinable()) t.join();
      c->fs = c->stream;
    }
  } far_join{c, far_thread};
  if (overlap && c->capture) {  // no host syncs inside: the far launches go inline on s2
    CUDA_TRY(c, cudaStreamWaitEvent(c->s2, ev[6], 0));
    c->fs = c->s2;
    far_rc = far_sum(c, T, txy, c->d_ufar.as<double>(), false);
    if (!far_rc) CUDA_TRY(c, cudaEventRecord(c->ev[2], c->s2));
  } else if (overlap) {
    CUDA_TRY(c, cudaStreamWaitEvent(c->s2, ev[6], 0));
    c->fs = c->s2;
    far_thread = std::thread([c, T, txy, &far_rc] {
      cudaSetDevice(c->device);
      far_rc = far_sum(c, T, txy, c->d_ufar.as<double>(), false);
      if (!far_rc && cudaEventRecord(c->ev[2], c->s2) != cudaSuccess) far_rc = set_err(c, 3, "cuda: far event");
    });
  } else if (c->far_method == 2) {
    // corrections only: the caller supplies the far field (subtract-and-add,
    // SPEC.md:612-615); u = sum over N(t) and S(t) of (I_T - point sum)
    CUDA_TRY(c, cudaMemsetAsync(c->d_ufar.p, 0, sizeof(double) * (T + 1), c->stream));
    CUDA_TRY(c, cudaEventRecord(ev[2], c->stream));
  } else {
    if (int rc = far_sum(c, T, txy, c->d_ufar.as<double>(), false)) return rc;
    CUDA_TRY(c, cudaEventRecord(ev[2], c->stream));
  }
  // Pair stage.  The self pairs and the per-target point sums need only the
  // lists and the sources, so they run on s3 beside the near chain (whose
  // leaf walk is latency-bound and whose host syncs would otherwise leave
  // the GPU idle); the main stream has the higher priority, so the near
  // chain's blocks go first and K5 fills the rest.
  CUDA_TRY(c, c->d_corr_self.ensure(sizeof(double) * (T + 1)));
  CUDA_TRY(c, c->d_psum.ensure(sizeof(double) * (T + 1)));
  const cudaEvent_t fork = overlap ? ev[6] : ev[2];
  struct SelfStream {  // launch_self goes to s3 until this scope ends
    vp_ctx* c;
    ~SelfStream() { c->ss = c->stream; }
  } self_stream{c};
  CUDA_TRY(c, cudaStreamWaitEvent(c->s3, fork, 0));
  c->ss = c->s3;
  VP_DISPATCH_P(c->p, launch_self, c, T, nullptr, c->d_self.as<int32_t>(), txy, c->d_corr_self.as<double>(),
                nullptr, nullptr);
  CUDA_TRY(c, cudaEventRecord(ev[9], c->s3));
  {
    const unsigned pblocks = (unsigned)std::min<int64_t>(nblk(T, PT_WARPS), (int64_t)c->sm_count * 64);
    auto psum_args = [&](auto kern, int copies) {
      kern<<<pblocks, PT_WARPS * 32, sizeof(double2) * kLogEntries * copies, c->s3>>>(
          T, txy, c->d_self.as<int32_t>(), c->d_off.as<int64_t>(), c->d_ids.as<int32_t>(), c->rules.len_q,
          c->d_sx.as<double>(), c->d_sy.as<double>(), c->d_sq.as<double>(), c->d_psum.as<double>(),
          (int64_t)c->n_tri * c->rules.len_q < (1ll << 32) ? 1 : 0);
    };
    switch (c->psum_copies) {
      case 2: psum_args(k_psum_tgt<2>, 2); break;
      case 8: psum_args(k_psum_tgt<8>, 8); break;
      case 4: psum_args(k_psum_tgt<4>, 4); break;
      default: psum_args(k_psum_tgt<1>, 1); break;
    }
  }
  CUDA_TRY(c, cudaEventRecord(ev[8], c->s3));
  c->ss = c->stream;
  c->last_launches += 2;
  CUDA_TRY(c, c->d_ptgt.ensure(sizeof(int32_t) * (n_ids + 1)));
  CUDA_TRY(c, c->d_corr.ensure(sizeof(double) * (n_ids + 1)));
  if (n_ids > 0) {
    k_pair_tgt<<<nblk(T, 256), 256, 0, c->stream>>>(T, c->d_off.as<int64_t>(), c->d_ptgt.as<int32_t>());
    c->last_launches += 1;
    if (int rc = launch_near(c, n_ids, c->d_ptgt.as<int32_t>(), c->d_ids.as<int32_t>(), txy,
                             c->d_corr.as<double>(), nullptr, nullptr, T, c->d_off.as<int64_t>())) return rc;
  }
  CUDA_TRY(c, cudaEventRecord(ev[3], c->stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, ev[8], 0));
  CUDA_TRY(c, cudaEventRecord(ev[4], c->stream));
  if (far_thread.joinable()) far_thread.join();
  c->fs = c->stream;
  if (far_rc) return far_rc;
  c->last_launches += c->far_launches;
  if (overlap) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, ev[2], 0));
  CUDA_TRY(c, c->d_neart.ensure(sizeof(double) * (T + 1)));
  k_assemble<<<nblk(T, 256), 256, 0, c->stream>>>(T, c->d_ufar.as<double>(), c->d_psum.as<double>(),
                                                   c->d_neart.as<double>(), c->d_off.as<int64_t>(),
                                                   c->d_corr.as<double>(), c->d_corr_self.as<double>(), u);
  k_count_self<<<nblk(T, 256), 256, 0, c->stream>>>(T, c->d_self.as<int32_t>(), c->d_stats.as<unsigned long long>());
  c->last_launches += 2;
  CUDA_TRY(c, cudaEventRecord(ev[5], c->stream));
  CUDA_TRY(c, cudaGetLastError());
  if (c->capture) {  // stats and error flags of every replay land in pinned memory
    CUDA_TRY(c, cudaMemcpyAsync(c->h_gstats, c->d_stats.p, sizeof(unsigned long long) * 8, cudaMemcpyDeviceToHost,
                                c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_gstats + 8, c->d_err.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    fork_guard.ok = true;
    return 0;
  }
  unsigned long long hs[8];
  int herr[2] = {0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(hs, c->d_stats.p, sizeof(hs), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(herr, c->d_err.p, sizeof(herr), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (herr[1]) return set_err(c, 2, "evaluate: non-finite target coordinate");
  if (herr[0]) return set_err(c, 2, "near_eval: subdivision exceeded depth/frontier limits "
                                    "(target effectively on element boundary)");
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->n_targets = T;
    st->n_near_pairs = n_ids;
    st->n_leaves = (n_ids > 0 ? c->n_leaves_last : 0) + (int64_t)hs[6];
    st->n_rho_le1 = (int64_t)hs[1];
    st->max_depth = (int32_t)hs[2];
    st->n_panels = (int64_t)hs[3];
    st->n_degenerate = (int64_t)hs[4];
    st->n_self = (int64_t)hs[5];
    st->n_outside = T - st->n_self;
    st->n_sources = c->n_tri * c->rules.len_q;
    st->gpu_launches = c->last_launches;
    st->far_method = c->far_method;
    st->fmm_levels = c->far_method == 1 ? c->fmm_levels : 0;
    st->fmm_outside = c->far_method == 1 ? c->fmm_outside : 0;
    float ms[2];
    for (int i = 0; i < 2; ++i) cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]);
    st->t_list_ms = ms[0];
    float msrc = 0, mfar = 0;
    cudaEventElapsedTime(&msrc, ev[1], ev[6]);
    cudaEventElapsedTime(&mfar, ev[6], ev[2]);
    st->t_sources_ms = msrc;
    st->t_far_kernel_ms = mfar;
    st->t_far_ms = ms[1];
    float mnear = 0, mself = 0, mpair = 0;
    cudaEventElapsedTime(&mnear, fork, ev[3]);  // with the FMM, near starts beside the far field
    cudaEventElapsedTime(&mself, fork, ev[9]);  // K5 on s3, beside the near chain
    cudaEventElapsedTime(&mpair, fork, ev[4]);  // near + self + point sums, overlapped
    st->t_near_ms = mnear;
    st->t_self_ms = mself;
    st->t_pair_ms = mpair;
    float tot = 0;
    cudaEventElapsedTime(&tot, ev[0], ev[5]);
    st->t_total_ms = tot;
  }
  fork_guard.ok = true;
  return 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
extern "C" {

const char* vp_last_error(const vp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int vp_create(int device, vp_ctx** out) {
  if (!out) return 1;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return 3;
  }
  if (device < 0 || device >= n) return 1;
  if (cudaSetDevice(device) != cudaSuccess) return 3;
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 3;
  if (prop.major < 10) return 3;  // sm_100a build only
  vp_ctx* c = new vp_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  if (const char* pc = std::getenv("VP_PSUM_COPIES")) c->psum_copies = std::atoi(pc);
  // k_psum_tgt<8> takes 64 KB of dynamic shared memory
  cudaFuncSetAttribute(k_psum_tgt<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(double2) * kLogEntries * 8));
  if (const char* lb = std::getenv("VP_LEAF_SCRATCH_BYTES")) {
    const long long v = std::atoll(lb);
    if (v > 0) c->leaf_scratch_budget = v;
  }
  // the main stream (lists, near chain) outranks s2 (FMM far) and s3 (self,
  // point sums), which fill the SMs the near chain leaves free
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (std::getenv("VP_FLAT_PRIO")) prio_hi = prio_lo;
  if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->s2, cudaStreamNonBlocking,
                                   std::getenv("VP_S2_HIGH") ? prio_hi : prio_lo) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->s3, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return 3;
  }
  c->fs = c->ss = c->stream;
  for (auto& e : c->ev) cudaEventCreate(&e);
  double cn[kMaxModes];
  for (int n2 = 0; n2 <= kMaxPdev; ++n2)
    for (int m = 0; m <= n2; ++m) cn[koorn_index(m, n2)] = std::sqrt((double)((2 * m + 1) * (2 * n2 + 2)));
  if (cudaFuncSetAttribute(k_far<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFarSmem) != cudaSuccess ||
      cudaFuncSetAttribute(k_far<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFarSmem) != cudaSuccess ||
      cudaFuncSetAttribute(k_far<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFarSmem) != cudaSuccess ||
      cudaFuncSetAttribute(k_far<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFarSmem) != cudaSuccess) {
    vp_destroy(c);
    return 3;
  }
  if (cudaFuncSetAttribute(k_near_c<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_ct<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_cg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_cg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_cg<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_cg<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_cg<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_cache_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)near_cache_mma_smem(kMaxModes)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_cache_mma2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)near_cache_mma2_smem(kMaxModes)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<0, self_gs(0)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(0)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<1, self_gs(1)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(1)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<2, self_gs(2)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(2)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<3, self_gs(3)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(3)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<4, self_gs(4)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(4)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<5, self_gs(5)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(5)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<6, self_gs(6)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(6)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<7, self_gs(7)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(7)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<8, self_gs(8)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(8)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<9, self_gs(9)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(9)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<10, self_gs(10)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(10)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<11, self_gs(11)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(11)) != cudaSuccess ||
      cudaFuncSetAttribute(k_self<12, self_gs(12)>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)self_dyn_smem(12)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<5, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<6, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<7, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_near_c8<8, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_fmm_eval<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_fmm_eval<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LogTab)) != cudaSuccess ||
      cudaFuncSetAttribute(k_fmm_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(k_fmm_m2m, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(k_fmm_p2m, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) {
    vp_destroy(c);
    return 3;
  }
  double2 lt[kLogEntries];
  log_table_fill(lt);
  std::vector<double2> ltf(kFarLogEntries);  // per call: vp_create may run on several threads
  log_table_fill(ltf.data(), kFarLogEntries);
  double la[kMaxCurveDeg + 1], lb[kMaxCurveDeg + 1];
  for (int k = 0; k <= kMaxCurveDeg; ++k) {
    la[k] = leg_la(k);
    lb[k] = leg_lb(k);
  }
  if (cudaMemcpyToSymbol(g_logtab, lt, sizeof(lt)) != cudaSuccess ||
      cudaMemcpyToSymbol(g_fartab, ltf.data(), sizeof(double2) * ltf.size()) != cudaSuccess ||
      cudaMemcpyToSymbol(c_cn, cn, sizeof(cn)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_leg_la, la, sizeof(la)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_leg_lb, lb, sizeof(lb)) != cudaSuccess) {
    vp_destroy(c);
    return 3;
  }
  *out = c;
  return 0;
}

void vp_destroy(vp_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->s2) cudaStreamDestroy(c->s2);
  if (c->s3) cudaStreamDestroy(c->s3);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->comm) vp_comm_release(c);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->h_gstats) cudaFreeHost(c->h_gstats);
  delete c;
}

int vp_set_near_model(vp_ctx* c, int model, double ball_factor) {
  if (!c) return 1;
  ++c->gen;
  if (model != 0 && model != 1) return set_err(c, 1, "set_near_model: model must be 0 (precise) or 1 (ball)");
  if (model == 1 && !(ball_factor >= 1.0)) return set_err(c, 1, "set_near_model: ball factor must be >= 1");
  c->near_model = model;
  c->ball_factor = model == 1 ? ball_factor : 1.5;
  if (c->have_rules) {
    c->h_rd.near_model = c->near_model;
    c->h_rd.ball_factor = c->ball_factor;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_rules.p, &c->h_rd, sizeof(RulesDev), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->have_mesh)
      if (int rc = build_elements(c)) return rc;
  }
  return 0;
}

int vp_set_near_cache(vp_ctx* c, int max_depth, int64_t max_bytes) {
  if (!c) return 1;
  ++c->gen;
  if (max_depth < -1 || max_depth > 6) return set_err(c, 1, "set_near_cache: max_depth must be in [-1, 6]");
  if (max_bytes < 0) return set_err(c, 1, "set_near_cache: max_bytes must be >= 0");
  c->cache_max_depth = max_depth;
  c->cache_max_bytes = max_bytes;  // 0: min(48 GiB, free / 4)
  return 0;
}

int vp_set_far_method(vp_ctx* c, int method, int order, int leaf_size) {
  if (!c) return 1;
  ++c->gen;
  if (method < 0 || method > 2)
    return set_err(c, 1, "set_far_method: method must be 0 (direct), 1 (fmm) or 2 (none: corrections only)");
  if (order != 0 && (order < 4 || order > kFmmMaxP))
    return set_err(c, 1, "set_far_method: FMM order must be in [4, 62] (0 = default 31)");
  if (leaf_size < 0) return set_err(c, 1, "set_far_method: leaf size must be >= 0 (0 = default 40)");
  c->far_method = method;
  c->fmm_p = order ? order : 31;  // p + 1 = 32 coefficients: one per lane
  c->fmm_leaf = leaf_size ? leaf_size : 40;
  return 0;
}

// eps_fmm -> expansion order.  The far-field error of the FMM
// against the direct sum, relative max-norm, measured on configs 1-4 by order
// (profiles/r02_fmm_order_sweep.json, tools/fmm_tolerance.py), stays below
// 0.15 * 0.41^p down to the rounding floor of 8e-15 at p = 31; the order is
// the smallest p with that bound <= eps_fmm, rounded up so that p + 1 is a
// multiple of four in [8, 32] (the orders k_fmm_m2l32 is instantiated for).
int vp_fmm_order_for(double eps_fmm) {
  if (!(eps_fmm > 0.0)) return 31;
  const double p = std::ceil(std::log(eps_fmm / 0.15) / std::log(0.41));
  int P1 = 4 * (int)std::ceil((std::max(p, 0.0) + 1.0) / 4.0);
  P1 = std::max(8, std::min(32, P1));
  return P1 - 1;
}

int vp_set_fmm_tolerance(vp_ctx* c, double eps_fmm, int leaf_size) {
  if (!c) return 1;
  if (!(eps_fmm > 0.0) || !(eps_fmm < 1.0))
    return set_err(c, 1, "set_fmm_tolerance: eps_fmm must be in (0, 1)");
  return vp_set_far_method(c, 1, vp_fmm_order_for(eps_fmm), leaf_size);
}

int vp_device_info(vp_ctx* c, int* sm_count, int* cc_major, int* cc_minor) {
  if (!c) return 1;
  cudaDeviceProp prop{};
  CUDA_TRY(c, cudaGetDeviceProperties(&prop, c->device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return 0;
}

int vp_set_mesh(vp_ctx* c, int64_t n_vert, const double* vxy, int64_t n_tri, const int32_t* tri) {
  if (!c) return 1;
  ++c->gen;
  if (n_vert <= 0 || n_tri <= 0 || !vxy || !tri)
    return set_err(c, 1, "set_mesh: empty mesh (invariant: n_vert > 0, n_tri > 0)");
  if (n_tri > (int64_t)INT32_MAX / 4) return set_err(c, 1, "set_mesh: too many triangles");
  for (int64_t i = 0; i < 3 * n_tri; ++i)
    if (tri[i] < 0 || tri[i] >= n_vert) return set_err(c, 1, "set_mesh: triangle vertex index out of range");
  for (int64_t i = 0; i < 2 * n_vert; ++i)
    if (!std::isfinite(vxy[i])) return set_err(c, 2, "set_mesh: non-finite vertex coordinate");
  c->h_vxy.assign(vxy, vxy + 2 * n_vert);
  c->h_tri.assign(tri, tri + 3 * n_tri);
  c->bx0 = c->by0 = 1e300;
  c->bx1 = c->by1 = -1e300;
  for (int64_t i = 0; i < n_vert; ++i) {
    c->bx0 = std::min(c->bx0, vxy[2 * i]);
    c->bx1 = std::max(c->bx1, vxy[2 * i]);
    c->by0 = std::min(c->by0, vxy[2 * i + 1]);
    c->by1 = std::max(c->by1, vxy[2 * i + 1]);
  }
  c->n_vert = n_vert;
  c->n_tri = n_tri;
  c->have_mesh = true;
  c->h_ecurve.clear();
  c->h_celist.clear();
  c->sources_valid = false;
  // triangle orientation is validated here so errors surface early
  for (int64_t e = 0; e < n_tri; ++e) {
    const int32_t* id = &tri[3 * e];
    const double e1x = vxy[2 * id[1]] - vxy[2 * id[0]], e1y = vxy[2 * id[1] + 1] - vxy[2 * id[0] + 1];
    const double e2x = vxy[2 * id[2]] - vxy[2 * id[0]], e2y = vxy[2 * id[2] + 1] - vxy[2 * id[0] + 1];
    const double t1 = e1x * e2y, t2 = e2x * e1y;
    if (!(t1 - t2 > 0.0)) {
      c->have_mesh = false;
      return set_err(c, 1, "set_mesh: triangle " + std::to_string(e) + " not counter-clockwise (invariant: det > 0)");
    }
  }
  if (c->have_rules) {
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (int rc = build_elements(c)) return rc;
  }
  if (c->have_density && c->M > 0) c->have_density = false;  // coefficients are per triangle
  return 0;
}

int vp_set_curves(vp_ctx* c, const int32_t* curve_id, int deg, int64_t n_curves, const double* cx,
                  const double* cy, const double* len) {
  if (!c) return 1;
  ++c->gen;
  if (!c->have_mesh) return set_err(c, 1, "set_curves: call vp_set_mesh first");
  c->h_ecurve.clear();
  c->h_celist.clear();
  c->sources_valid = false;
  if (curve_id) {
    if (deg < 1 || deg > 64) return set_err(c, 1, "set_curves: degree must be in [1, 64]");
    if (n_curves <= 0 || !cx || !cy || !len) return set_err(c, 1, "set_curves: empty curve arrays");
    for (int64_t i = 0; i < n_curves; ++i)
      if (!(len[i] > 0.0) || !std::isfinite(len[i])) return set_err(c, 1, "set_curves: arc length must be > 0");
    for (int64_t i = 0; i < n_curves * (deg + 1); ++i)
      if (!std::isfinite(cx[i]) || !std::isfinite(cy[i])) return set_err(c, 2, "set_curves: non-finite coefficient");
    std::vector<int32_t> ec(curve_id, curve_id + c->n_tri);
    std::vector<int32_t> cl;
    for (int64_t e = 0; e < c->n_tri; ++e) {
      if (ec[e] < -1 || ec[e] >= n_curves) return set_err(c, 1, "set_curves: curve id out of range");
      if (ec[e] >= 0) cl.push_back((int32_t)e);
    }
    if (!cl.empty()) {
      c->curve_deg = deg;
      c->h_ecurve = std::move(ec);
      c->h_celist = std::move(cl);
      c->h_ccx.assign(cx, cx + n_curves * (deg + 1));
      c->h_ccy.assign(cy, cy + n_curves * (deg + 1));
      c->h_clen.assign(len, len + n_curves);
      CUDA_TRY(c, cudaSetDevice(c->device));
      CUDA_TRY(c, c->d_ecurve.ensure(sizeof(int32_t) * c->n_tri));
      CUDA_TRY(c, c->d_celist.ensure(sizeof(int32_t) * c->h_celist.size()));
      CUDA_TRY(c, c->d_ccx.ensure(sizeof(double) * c->h_ccx.size()));
      CUDA_TRY(c, c->d_ccy.ensure(sizeof(double) * c->h_ccy.size()));
      CUDA_TRY(c, c->d_clen.ensure(sizeof(double) * n_curves));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_ecurve.p, c->h_ecurve.data(), sizeof(int32_t) * c->n_tri,
                                  cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_celist.p, c->h_celist.data(), sizeof(int32_t) * c->h_celist.size(),
                                  cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_ccx.p, c->h_ccx.data(), sizeof(double) * c->h_ccx.size(),
                                  cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_ccy.p, c->h_ccy.data(), sizeof(double) * c->h_ccy.size(),
                                  cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_clen.p, c->h_clen.data(), sizeof(double) * n_curves, cudaMemcpyHostToDevice,
                                  c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
  }
  if (c->have_rules) {
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (int rc = build_elements(c)) return rc;
  }
  return 0;
}

int vp_set_rules(vp_ctx* c, const vp_rules* r) {
  if (!c) return 1;
  ++c->gen;
  if (!r) return set_err(c, 1, "set_rules: null rules");
  if (r->len_q <= 0 || r->len_q > kMaxFar || !r->far_x || !r->far_y || !r->far_w)
    return set_err(c, 1, "set_rules: far rule length must be in [1, 1024]");
  if (r->len_n <= 0 || r->len_n > kMaxNearRule || !r->near_x || !r->near_y || !r->near_w)
    return set_err(c, 1, "set_rules: near rule length must be in [1, 256]");
  if (r->n_l <= 0 || r->n_l > kMaxGL || !r->gl_x || !r->gl_w)
    return set_err(c, 1, "set_rules: Gauss-Legendre length must be in [1, 64]");
  if (r->n_g < 0 || r->n_g + 1 > kMaxGGQ || !r->ggq_r || !r->ggq_w)
    return set_err(c, 1, "set_rules: GGQ order must be in [0, 31]");
  if (!(r->eps > 0.0) || r->q < 1 || r->n_n < 1) return set_err(c, 1, "set_rules: eps > 0, q >= 1, n_n >= 1 required");
  for (int i = 0; i < r->len_q; ++i)
    if (!(r->far_w[i] > 0.0)) return set_err(c, 2, "rule table: non-positive weight (invariant: weights > 0)");
  for (int i = 0; i <= r->n_g; ++i)
    if (!(r->ggq_r[i] > 0.0 && r->ggq_r[i] < 1.0)) return set_err(c, 2, "set_rules: GGQ nodes must lie in (0,1)");
  // keep host copies (the vp_rules pointers are caller-owned)
  std::vector<double>& st = c->h_rules_store;
  st.clear();
  auto keep = [&](const double* p, int n) {
    const size_t o = st.size();
    st.insert(st.end(), p, p + n);
    return o;
  };
  const size_t o1 = keep(r->far_x, r->len_q), o2 = keep(r->far_y, r->len_q), o3 = keep(r->far_w, r->len_q);
  const size_t o4 = keep(r->near_x, r->len_n), o5 = keep(r->near_y, r->len_n), o6 = keep(r->near_w, r->len_n);
  const size_t o7 = keep(r->gl_x, r->n_l), o8 = keep(r->gl_w, r->n_l);
  const size_t o9 = keep(r->ggq_r, r->n_g + 1), o10 = keep(r->ggq_w, r->n_g + 1);
  c->rules = *r;
  c->rules.far_x = &st[o1]; c->rules.far_y = &st[o2]; c->rules.far_w = &st[o3];
  c->rules.near_x = &st[o4]; c->rules.near_y = &st[o5]; c->rules.near_w = &st[o6];
  c->rules.gl_x = &st[o7]; c->rules.gl_w = &st[o8];
  c->rules.ggq_r = &st[o9]; c->rules.ggq_w = &st[o10];
  RulesDev& d = c->h_rd;
  std::memset(&d, 0, sizeof(d));
  d.len_q = r->len_q; d.len_n = r->len_n; d.n_l = r->n_l; d.n_g1 = r->n_g + 1; d.n_n = r->n_n; d.q = r->q;
  d.near_model = c->near_model;
  d.ball_factor = c->ball_factor;
  for (int i = 0; i < r->len_q; ++i) { d.far_x[i] = r->far_x[i]; d.far_y[i] = r->far_y[i]; d.far_w[i] = r->far_w[i]; }
  for (int i = 0; i < r->len_n; ++i) { d.near_x[i] = r->near_x[i]; d.near_y[i] = r->near_y[i]; d.near_w[i] = r->near_w[i]; }
  for (int i = 0; i < r->n_l; ++i) { d.gl_x[i] = r->gl_x[i]; d.gl_w[i] = r->gl_w[i]; }
  for (int i = 0; i <= r->n_g; ++i) { d.ggq_r[i] = r->ggq_r[i]; d.ggq_w[i] = r->ggq_w[i]; d.ggq_lr[i] = std::log(r->ggq_r[i]); }
  for (int k = 0; k <= kMaxNearDepth + 1; ++k) d.kd[k] = std::pow(4.0, -(double)k / (double)r->n_n);
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, c->d_rules.ensure(sizeof(RulesDev)));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_rules.p, &d, sizeof(RulesDev), cudaMemcpyHostToDevice, c->stream));
  c->have_rules = true;
  c->sources_valid = false;
  c->cacheV_depth = -2;
  c->tabs_p = -1;
  if (c->have_mesh)
    if (int rc = build_elements(c)) return rc;
  if (int rc = upload_self_tab(c)) return rc;
  if (c->p >= 0) {  // Koornwinder values at the far nodes for K1
    const int M = koorn_size(c->p);
    std::vector<double> V((size_t)r->len_q * M);
    for (int i = 0; i < r->len_q; ++i) koorn_eval(c->p, r->far_x[i], r->far_y[i], &V[(size_t)i * M]);
    CUDA_TRY(c, c->d_V.ensure(sizeof(double) * V.size()));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_V.p, V.data(), sizeof(double) * V.size(), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->tabs_p = c->p;
  }
  return 0;
}

int vp_set_density(vp_ctx* c, int p, const double* coeffs) {
  if (!c) return 1;
  if (!c->have_mesh) return set_err(c, 1, "usage: vp_set_mesh must precede vp_set_density");
  if (p < 0 || p > kMaxPdev) return set_err(c, 1, "set_density: order p must be in [0, 12]");
  if (!coeffs) return set_err(c, 1, "set_density: null coefficients");
  const int M = koorn_size(p);
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (p != c->p || c->d_coeffs.cap < sizeof(double) * c->n_tri * M) ++c->gen;  // a captured graph reads d_coeffs
  CUDA_TRY(c, c->d_coeffs.ensure(sizeof(double) * c->n_tri * M));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_coeffs.p, coeffs, sizeof(double) * c->n_tri * M, cudaMemcpyHostToDevice, c->stream));
  c->p = p;
  c->M = M;
  c->have_density = true;
  c->sources_valid = false;
  // K1's Koornwinder table, the near-cache Vt and the SelfTab depend on (p,
  // rules) only: a new density of the same order reuses them
  if (c->have_rules && c->tabs_p == p) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return 0;
  }
  if (c->have_rules) {
    const vp_rules& r = c->rules;
    std::vector<double> V((size_t)r.len_q * M);
    for (int i = 0; i < r.len_q; ++i) koorn_eval(p, r.far_x[i], r.far_y[i], &V[(size_t)i * M]);
    CUDA_TRY(c, c->d_V.ensure(sizeof(double) * V.size()));
    CUDA_TRY(c, cudaMemcpyAsync(c->d_V.p, V.data(), sizeof(double) * V.size(), cudaMemcpyHostToDevice, c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->cacheV_depth = -2;
  if (int rc = upload_self_tab(c)) return rc;
  c->tabs_p = c->have_rules ? p : -1;
  return 0;
}

int vp_build_nearlist(vp_ctx* c, int64_t n_tgt, const double* txy, int32_t* self_out, int64_t* offsets_out,
                      int32_t* ids_out, int64_t ids_cap, int64_t* n_ids) {
  if (int rc = ensure_ready(c, false)) return rc;
  if (n_tgt < 0 || (n_tgt > 0 && !txy)) return set_err(c, 1, "nearlist: bad target array");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (n_tgt == 0) {
    if (offsets_out) offsets_out[0] = 0;
    if (n_ids) *n_ids = 0;
    return 0;
  }
  CUDA_TRY(c, c->d_txy.ensure(sizeof(double) * 2 * n_tgt));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_txy.p, txy, sizeof(double) * 2 * n_tgt, cudaMemcpyHostToDevice, c->stream));
  int64_t nids = 0;
  if (int rc = build_lists(c, n_tgt, c->d_txy.as<double2>(), &nids)) return rc;
  if (n_ids) *n_ids = nids;
  if (self_out)
    CUDA_TRY(c, cudaMemcpyAsync(self_out, c->d_self.p, sizeof(int32_t) * n_tgt, cudaMemcpyDeviceToHost, c->stream));
  if (offsets_out)
    CUDA_TRY(c, cudaMemcpyAsync(offsets_out, c->d_off.p, sizeof(int64_t) * (n_tgt + 1), cudaMemcpyDeviceToHost, c->stream));
  if (ids_out) {
    if (nids > ids_cap) {
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      return set_err(c, 1, "nearlist: ids capacity too small");
    }
    if (nids > 0)
      CUDA_TRY(c, cudaMemcpyAsync(ids_out, c->d_ids.p, sizeof(int32_t) * nids, cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return 0;
}

int vp_evaluate_device(vp_ctx* c, int64_t n_tgt, const double* d_txy, double* d_u, void* stream, vp_stats* st) {
  if (int rc = ensure_ready(c, true)) return rc;
  if (n_tgt < 0 || (n_tgt > 0 && (!d_txy || !d_u))) return set_err(c, 1, "evaluate: bad target array");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (n_tgt == 0) {
    if (st) std::memset(st, 0, sizeof(*st));
    return 0;
  }
  cudaStream_t user = (cudaStream_t)stream;
  if (user) {  // order against the caller's stream
    cudaEvent_t e;
    CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEventRecord(e, user);
    cudaStreamWaitEvent(c->stream, e, 0);
    cudaEventDestroy(e);
  }
  const int rc = evaluate_impl(c, n_tgt, (const double2*)d_txy, d_u, st);
  return rc;
}

int vp_evaluate_graph(vp_ctx* c, int64_t n_tgt, const double* d_txy, double* d_u, void* stream) {
  if (int rc = ensure_ready(c, true)) return rc;
  if (n_tgt <= 0 || !d_txy || !d_u) return set_err(c, 1, "evaluate_graph: need n_tgt > 0 and device arrays");
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaStream_t user = stream ? (cudaStream_t)stream : c->stream;
  const bool fresh = c->gexec && c->g_gen == c->gen && c->g_n == n_tgt && c->g_txy == d_txy && c->g_u == d_u;
  if (!fresh) {
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->graph) cudaGraphDestroy(c->graph);
    c->gexec = nullptr;
    c->graph = nullptr;
    if (!c->h_gstats) CUDA_TRY(c, cudaMallocHost(&c->h_gstats, sizeof(unsigned long long) * 16));
    // eager evaluation on the ctx stream: fills the plan and every buffer
    if (user != c->stream) {
      cudaEvent_t e;
      CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      cudaEventRecord(e, user);
      cudaStreamWaitEvent(c->stream, e, 0);
      cudaEventDestroy(e);
    }
    if (int rc = evaluate_impl(c, n_tgt, (const double2*)d_txy, d_u, nullptr)) return rc;
    // capture the same evaluation with the plan's sizes
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->capture = true;
    const int rc = evaluate_impl(c, n_tgt, (const double2*)d_txy, d_u, nullptr);
    c->capture = false;
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return set_err(c, 3, std::string("cuda: capture failed: ") + cudaGetErrorString(ce));
    CUDA_TRY(c, cudaGraphInstantiate(&c->gexec, g, 0));
    c->graph = g;
    c->g_gen = c->gen;
    c->g_n = n_tgt;
    c->g_txy = d_txy;
    c->g_u = d_u;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  }
  CUDA_TRY(c, cudaGraphLaunch(c->gexec, user));
  return 0;
}

int vp_graph_status(vp_ctx* c, void* stream, vp_stats* st) {
  if (!c) return 1;
  if (!c->gexec) return set_err(c, 1, "graph_status: no captured evaluation");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(stream ? (cudaStream_t)stream : c->stream));
  const unsigned long long* hs = c->h_gstats;
  const int* herr = reinterpret_cast<const int*>(hs + 8);
  if (herr[1]) return set_err(c, 2, "evaluate: non-finite target coordinate");
  if (herr[0]) return set_err(c, 2, "near_eval: subdivision exceeded depth/frontier limits");
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->n_targets = c->g_n;
    st->n_near_pairs = c->plan.n_ids;
    st->n_leaves = c->plan.tot0 + c->plan.tot1 + (int64_t)hs[6];
    st->n_rho_le1 = (int64_t)hs[1];
    st->max_depth = (int32_t)hs[2];
    st->n_panels = (int64_t)hs[3];
    st->n_degenerate = (int64_t)hs[4];
    st->n_self = (int64_t)hs[5];
    st->n_outside = c->g_n - st->n_self;
    st->n_sources = c->n_tri * c->rules.len_q;
    st->far_method = c->far_method;
  }
  return 0;
}

int vp_evaluate(vp_ctx* c, int64_t n_tgt, const double* txy, double* u_out, vp_stats* st) {
  if (int rc = ensure_ready(c, true)) return rc;
  if (n_tgt < 0 || (n_tgt > 0 && (!txy || !u_out))) return set_err(c, 1, "evaluate: bad target array");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (n_tgt == 0) {
    if (st) std::memset(st, 0, sizeof(*st));
    return 0;
  }
  CUDA_TRY(c, c->d_txy.ensure(sizeof(double) * 2 * n_tgt));
  CUDA_TRY(c, c->d_u.ensure(sizeof(double) * n_tgt));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_txy.p, txy, sizeof(double) * 2 * n_tgt, cudaMemcpyHostToDevice, c->stream));
  if (int rc = evaluate_impl(c, n_tgt, c->d_txy.as<double2>(), c->d_u.as<double>(), st)) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(u_out, c->d_u.p, sizeof(double) * n_tgt, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return 0;
}

int vp_far_field(vp_ctx* c, int64_t n_tgt, const double* txy, double* u_far) {
  if (int rc = ensure_ready(c, true)) return rc;
  if (n_tgt <= 0 || !txy || !u_far) return set_err(c, 1, "far_field: bad target array");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, c->d_txy.ensure(sizeof(double) * 2 * n_tgt));
  CUDA_TRY(c, c->d_ufar.ensure(sizeof(double) * n_tgt));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_txy.p, txy, sizeof(double) * 2 * n_tgt, cudaMemcpyHostToDevice, c->stream));
  if (int rc = compute_sources(c)) return rc;
  if (int rc = far_sum(c, n_tgt, c->d_txy.as<double2>(), c->d_ufar.as<double>(), true)) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(u_far, c->d_ufar.p, sizeof(double) * n_tgt, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return 0;
}

int vp_sources(vp_ctx* c, double* sx, double* sy, double* q) {
  if (int rc = ensure_ready(c, true)) return rc;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (int rc = compute_sources(c)) return rc;
  const size_t n = sizeof(double) * c->n_tri * c->rules.len_q;
  if (sx) CUDA_TRY(c, cudaMemcpyAsync(sx, c->d_sx.p, n, cudaMemcpyDeviceToHost, c->stream));
  if (sy) CUDA_TRY(c, cudaMemcpyAsync(sy, c->d_sy.p, n, cudaMemcpyDeviceToHost, c->stream));
  if (q) CUDA_TRY(c, cudaMemcpyAsync(q, c->d_sq.p, n, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return 0;
}

static int pairs_common(vp_ctx* c, int64_t n, const double* txy, const int32_t* elem, bool self,
                        double* val, double* sub, int64_t* cnt) {
  if (int rc = ensure_ready(c, true)) return rc;
  if (n <= 0 || !txy || !elem || !val) return set_err(c, 1, "pairs: bad arrays");
  for (int64_t i = 0; i < n; ++i)
    if (elem[i] < 0 || elem[i] >= c->n_tri) return set_err(c, 1, "pairs: element out of range");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (int rc = compute_sources(c)) return rc;
  CUDA_TRY(c, c->d_stats.ensure(sizeof(unsigned long long) * 8));
  CUDA_TRY(c, c->d_err.ensure(2 * sizeof(int)));
  CUDA_TRY(c, cudaMemsetAsync(c->d_stats.p, 0, sizeof(unsigned long long) * 8, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(c->d_err.p, 0, 2 * sizeof(int), c->stream));
  CUDA_TRY(c, c->d_txy.ensure(sizeof(double) * 2 * n));
  CUDA_TRY(c, c->d_pelem.ensure(sizeof(int32_t) * n));
  CUDA_TRY(c, c->d_ptgt.ensure(sizeof(int32_t) * n));
  CUDA_TRY(c, c->d_corr.ensure(sizeof(double) * n));
  CUDA_TRY(c, c->d_sub.ensure(sizeof(double) * n));
  CUDA_TRY(c, c->d_leaves.ensure(sizeof(int64_t) * n));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_txy.p, txy, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_pelem.p, elem, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
  std::vector<int32_t> idx(n);
  for (int64_t i = 0; i < n; ++i) idx[i] = (int32_t)i;
  CUDA_TRY(c, cudaMemcpyAsync(c->d_ptgt.p, idx.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
  if (self) {
    VP_DISPATCH_P(c->p, launch_self, c, n, c->d_ptgt.as<int32_t>(), c->d_pelem.as<int32_t>(),
                  c->d_txy.as<double2>(), c->d_corr.as<double>(), c->d_sub.as<double>(), c->d_leaves.as<int64_t>());
  } else {
    if (int rc = launch_near(c, n, c->d_ptgt.as<int32_t>(), c->d_pelem.as<int32_t>(), c->d_txy.as<double2>(),
                             c->d_corr.as<double>(), c->d_sub.as<double>(), nullptr)) return rc;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_leaves.p, c->d_lcnt.p, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c->stream));
  }
  CUDA_TRY(c, cudaGetLastError());
  int herr = 0;
  CUDA_TRY(c, cudaMemcpyAsync(val, c->d_corr.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  if (sub) CUDA_TRY(c, cudaMemcpyAsync(sub, c->d_sub.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  if (cnt) CUDA_TRY(c, cudaMemcpyAsync(cnt, c->d_leaves.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(&herr, c->d_err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (herr) return set_err(c, 2, "near_eval: subdivision exceeded depth/frontier limits");
  return 0;
}

// interp_coeffs (rules.hpp:165-170) batched on the device: the inverse
// Vandermonde of the interpolation nodes is formed on the host by Gauss-Jordan
// elimination with partial pivoting (make_interp_rule, rules.hpp:139-156).
int vp_interp_coeffs(vp_ctx* c, int p, const double* ref_x, const double* ref_y, int64_t n_elem,
                     const double* values, double* coeffs, double* cond) {
  if (!c) return 1;
  if (p < 0 || p > kMaxPdev) return set_err(c, 1, "interp_coeffs: order p must be in [0, 12]");
  if (n_elem <= 0 || !ref_x || !ref_y || !values || !coeffs)
    return set_err(c, 1, "interp_coeffs: value count must equal rule length (empty input)");
  const int M = koorn_size(p);
  std::vector<double> V((size_t)M * M), A((size_t)M * 2 * M, 0.0);
  for (int i = 0; i < M; ++i) {
    if (ref_x[i] < -1e-9 || ref_y[i] < -1e-9 || ref_x[i] + ref_y[i] > 1 + 1e-9)
      return set_err(c, 2, "interp_coeffs: node outside the simplex");
    koorn_eval(p, ref_x[i], ref_y[i], &V[(size_t)i * M]);
  }
  for (int i = 0; i < M; ++i) {
    for (int j = 0; j < M; ++j) A[(size_t)i * 2 * M + j] = V[(size_t)i * M + j];
    A[(size_t)i * 2 * M + M + i] = 1.0;
  }
  for (int col = 0; col < M; ++col) {
    int piv = col;
    for (int r = col + 1; r < M; ++r)
      if (std::abs(A[(size_t)r * 2 * M + col]) > std::abs(A[(size_t)piv * 2 * M + col])) piv = r;
    if (!(std::abs(A[(size_t)piv * 2 * M + col]) > 0.0))
      return set_err(c, 2, "interp_coeffs: nodes are not unisolvent (singular Vandermonde)");
    if (piv != col)
      for (int k = 0; k < 2 * M; ++k) std::swap(A[(size_t)col * 2 * M + k], A[(size_t)piv * 2 * M + k]);
    const double d = A[(size_t)col * 2 * M + col];
    for (int k = 0; k < 2 * M; ++k) A[(size_t)col * 2 * M + k] /= d;
    for (int r = 0; r < M; ++r) {
      if (r == col) continue;
      const double f = A[(size_t)r * 2 * M + col];
      if (f == 0.0) continue;
      for (int k = 0; k < 2 * M; ++k) A[(size_t)r * 2 * M + k] -= f * A[(size_t)col * 2 * M + k];
    }
  }
  std::vector<double> Vinv((size_t)M * M);
  double nv = 0.0, ni = 0.0;  // infinity-norm condition number estimate
  for (int i = 0; i < M; ++i) {
    double rv = 0.0, ri = 0.0;
    for (int j = 0; j < M; ++j) {
      Vinv[(size_t)i * M + j] = A[(size_t)i * 2 * M + M + j];
      rv += std::abs(V[(size_t)i * M + j]);
      ri += std::abs(Vinv[(size_t)i * M + j]);
    }
    nv = std::max(nv, rv);
    ni = std::max(ni, ri);
  }
  if (cond) *cond = nv * ni;
  CUDA_TRY(c, cudaSetDevice(c->device));
  DevBuf dV, dvals, dout;
  CUDA_TRY(c, dV.ensure(sizeof(double) * Vinv.size()));
  CUDA_TRY(c, dvals.ensure(sizeof(double) * n_elem * M));
  CUDA_TRY(c, dout.ensure(sizeof(double) * n_elem * M));
  CUDA_TRY(c, cudaMemcpyAsync(dV.p, Vinv.data(), sizeof(double) * Vinv.size(), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dvals.p, values, sizeof(double) * n_elem * M, cudaMemcpyHostToDevice, c->stream));
  k_interp<<<nblk(n_elem, kCacheNE), 128, 0, c->stream>>>(n_elem, M, dV.as<double>(), dvals.as<double>(),
                                                          dout.as<double>());
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaMemcpyAsync(coeffs, dout.p, sizeof(double) * n_elem * M, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return 0;
}

extern "C++" {
template <int P>
void launch_field_eval(vp_ctx* c, int64_t n, const double2* pts, const TriBox* tb, const double4* bb, GridDev g,
                       const int64_t* cb, const int64_t* ce, const int32_t* cel, const double* coeffs, double* out,
                       int32_t* eo) {
  k_field_eval<P><<<nblk(n, 128), 128, 0, c->stream>>>(n, pts, tb, bb, g, cb, ce, cel, coeffs, out, eo);
}
}

int vp_field_eval(vp_ctx* c, int64_t n_vert, const double* vxy, int64_t n_tri, const int32_t* tri, int p,
                  const double* coeffs, int64_t n_pts, const double* pts, double* out, int32_t* elem_out,
                  int64_t* n_outside) {
  if (!c) return 1;
  if (n_vert <= 0 || n_tri <= 0 || !vxy || !tri) return set_err(c, 1, "field_eval: empty interpolation mesh");
  if (p < 0 || p > kMaxPdev || !coeffs) return set_err(c, 1, "field_eval: order p must be in [0, 12]");
  if (n_pts < 0 || (n_pts > 0 && (!pts || !out))) return set_err(c, 1, "field_eval: bad point array");
  for (int64_t i = 0; i < 3 * n_tri; ++i)
    if (tri[i] < 0 || tri[i] >= n_vert) return set_err(c, 1, "field_eval: triangle vertex index out of range");
  if (n_pts == 0) {
    if (n_outside) *n_outside = 0;
    return 0;
  }
  const int M = koorn_size(p);
  CUDA_TRY(c, cudaSetDevice(c->device));
  DevBuf dv, dt, dtb, dbb, dcf, dp, dout, deo, cnt, off, keys, vals, keys2, cel, cb, ce;
  CUDA_TRY(c, dv.ensure(sizeof(double) * 2 * n_vert));
  CUDA_TRY(c, dt.ensure(sizeof(int32_t) * 3 * n_tri));
  CUDA_TRY(c, dtb.ensure(sizeof(TriBox) * n_tri));
  CUDA_TRY(c, dbb.ensure(sizeof(double4) * n_tri));
  CUDA_TRY(c, dcf.ensure(sizeof(double) * n_tri * M));
  CUDA_TRY(c, dp.ensure(sizeof(double) * 2 * n_pts));
  CUDA_TRY(c, dout.ensure(sizeof(double) * n_pts));
  CUDA_TRY(c, deo.ensure(sizeof(int32_t) * n_pts));
  CUDA_TRY(c, cudaMemcpyAsync(dv.p, vxy, sizeof(double) * 2 * n_vert, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dt.p, tri, sizeof(int32_t) * 3 * n_tri, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dcf.p, coeffs, sizeof(double) * n_tri * M, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dp.p, pts, sizeof(double) * 2 * n_pts, cudaMemcpyHostToDevice, c->stream));
  k_tri_boxes<<<nblk(n_tri, 256), 256, 0, c->stream>>>(n_tri, dv.as<double2>(), dt.as<int32_t>(), dtb.as<TriBox>(),
                                                        dbb.as<double4>());
  // grid: cell = mean triangle extent, from the mesh bounding box (host)
  double gx0 = 1e300, gy0 = 1e300, gx1 = -1e300, gy1 = -1e300;
  for (int64_t i = 0; i < n_vert; ++i) {
    gx0 = std::min(gx0, vxy[2 * i]);
    gx1 = std::max(gx1, vxy[2 * i]);
    gy0 = std::min(gy0, vxy[2 * i + 1]);
    gy1 = std::max(gy1, vxy[2 * i + 1]);
  }
  const double W = gx1 - gx0, H = gy1 - gy0;
  GridDev g;
  g.cs = std::max(std::sqrt(std::max(W * H, 1e-300) / (double)n_tri) * 1.5, 1e-300);
  while ((W / g.cs + 1) * (H / g.cs + 1) > double(1 << 24)) g.cs *= 1.5;
  g.x0 = gx0 - 1e-9 * (W + H);
  g.y0 = gy0 - 1e-9 * (W + H);
  g.nx = std::max(1, (int)std::ceil((W + 2e-9 * (W + H)) / g.cs));
  g.ny = std::max(1, (int)std::ceil((H + 2e-9 * (W + H)) / g.cs));
  g.inv_cs = 1.0 / g.cs;
  const int64_t ncell = (int64_t)g.nx * g.ny;
  CUDA_TRY(c, cnt.ensure(sizeof(int64_t) * (n_tri + 1)));
  CUDA_TRY(c, off.ensure(sizeof(int64_t) * (n_tri + 1)));
  k_box_count<<<nblk(n_tri, 256), 256, 0, c->stream>>>(n_tri, dbb.as<double4>(), g, cnt.as<int64_t>());
  CUDA_TRY(c, cudaMemsetAsync(cnt.as<int64_t>() + n_tri, 0, sizeof(int64_t), c->stream));
  size_t tmpb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmpb, cnt.as<int64_t>(), off.as<int64_t>(), n_tri + 1, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceScan::ExclusiveSum(c->d_tmp.p, tmpb, cnt.as<int64_t>(), off.as<int64_t>(), n_tri + 1, c->stream);
  int64_t np = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&np, off.as<int64_t>() + n_tri, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  CUDA_TRY(c, keys.ensure(sizeof(int32_t) * (np + 1)));
  CUDA_TRY(c, vals.ensure(sizeof(int32_t) * (np + 1)));
  CUDA_TRY(c, keys2.ensure(sizeof(int32_t) * (np + 1)));
  CUDA_TRY(c, cel.ensure(sizeof(int32_t) * (np + 1)));
  CUDA_TRY(c, cb.ensure(sizeof(int64_t) * ncell));
  CUDA_TRY(c, ce.ensure(sizeof(int64_t) * ncell));
  k_box_fill<<<nblk(n_tri, 256), 256, 0, c->stream>>>(n_tri, dbb.as<double4>(), g, off.as<int64_t>(),
                                                       keys.as<int32_t>(), vals.as<int32_t>());
  int endbit = 1;
  while ((1ll << endbit) < ncell) ++endbit;
  tmpb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmpb, keys.as<int32_t>(), keys2.as<int32_t>(), vals.as<int32_t>(),
                                  cel.as<int32_t>(), (int)np, 0, endbit, c->stream);
  CUDA_TRY(c, c->d_tmp.ensure(tmpb));
  cub::DeviceRadixSort::SortPairs(c->d_tmp.p, tmpb, keys.as<int32_t>(), keys2.as<int32_t>(), vals.as<int32_t>(),
                                  cel.as<int32_t>(), (int)np, 0, endbit, c->stream);
  CUDA_TRY(c, cudaMemsetAsync(cb.p, 0, sizeof(int64_t) * ncell, c->stream));
  CUDA_TRY(c, cudaMemsetAsync(ce.p, 0, sizeof(int64_t) * ncell, c->stream));
  if (np > 0)
    k_cell_ranges<<<nblk(np, 256), 256, 0, c->stream>>>(np, keys2.as<int32_t>(), cb.as<int64_t>(), ce.as<int64_t>());
  VP_DISPATCH_P(p, launch_field_eval, c, n_pts, dp.as<double2>(), dtb.as<TriBox>(), dbb.as<double4>(), g,
                cb.as<int64_t>(), ce.as<int64_t>(), cel.as<int32_t>(), dcf.as<double>(), dout.as<double>(),
                deo.as<int32_t>());
  CUDA_TRY(c, cudaGetLastError());
  std::vector<int32_t> eo(n_pts);
  CUDA_TRY(c, cudaMemcpyAsync(out, dout.p, sizeof(double) * n_pts, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(eo.data(), deo.p, sizeof(int32_t) * n_pts, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  int64_t nout = 0;
  for (int64_t i = 0; i < n_pts; ++i) nout += eo[i] < 0;
  if (elem_out) std::memcpy(elem_out, eo.data(), sizeof(int32_t) * n_pts);
  if (n_outside) *n_outside = nout;
  return 0;
}

int vp_near_pairs(vp_ctx* c, int64_t n, const double* txy, const int32_t* elem, double* val, double* sub,
                  int64_t* leaves) {
  return pairs_common(c, n, txy, elem, false, val, sub, leaves);
}

int vp_self_pairs(vp_ctx* c, int64_t n, const double* txy, const int32_t* elem, double* val, double* sub,
                  int64_t* panels) {
  return pairs_common(c, n, txy, elem, true, val, sub, panels);
}

}  // extern "C"

#include "vp_multi.cuh"
