// vp_fmm.cuh -- 2-D Laplace fast multipole method for the far field
// (SURVEY.md §8(f1)).
//
// Included by vp_b200.cu (one translation unit).  Computes the same quantity
// as K2 k_far, u_far[t] = sum_j q_j log|z_t - z_j|^2 = 2 Re sum_j q_j log(z_t - z_j),
// to the expansion accuracy instead of O(T S):
//   uniform quadtree over the sources (root = source bbox + margin, so the tree
//   and every u(t) are independent of the target set / sharding);
//   complex multipole and local expansions of order p, scaled by the box size
//   so every translation operator is O(1) and level independent;
//   P2M, M2M (upward), M2L over the classic interaction list + L2L
//   (downward), L2P + P2P with the 3x3 neighbour leaves (direct, fast log).
// Every reduction has a fixed order: results are bitwise reproducible.
//
// Translation formulas (Greengard & Rokhlin, Lemmas 2.3-2.5), in scaled form
// (a_k = â_k h^k about a box of size h; local b_l = b̂_l / h^l):
//   P2M  â_k = -sum q_j w_j^k / k,  w_j = (z_j - c)/h,  Q = sum q_j
//   M2M  b̂_l = -Q d^l / l + sum_{k=1}^{l} â_k 2^{-k} d^{l-k} C(l-1,k-1),  d = (c_child - c_par)/h_par
//   M2L  e_k = â_k (-1/D)^k;  b̂_0 += Q log(h|D|) + sum_k e_k;
//        b̂_l += D^{-l} (-Q/l + sum_k C(l+k-1,k-1) e_k),  D = (c_src - c_tgt)/h
//   L2L  b̂'_l = 2^{-l} sum_{k>=l} b̂_k C(k,l) d^{k-l},  d = (c_child - c_par)/h_par
//   L2P  Phi(z) = sum_l b̂_l eta^l,  eta = (z - c)/h
// The imaginary part of the log term never reaches Re Phi, so only its real
// part Q log(h|D|) is accumulated.

constexpr int kFmmMaxP = 62;  // p + 1 <= 63 coefficients: two per lane
constexpr int kFmmThreads = 128;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma_r(double r, double2 a, double2 acc) {  // acc + r a
  return make_double2(fma(r, a.x, acc.x), fma(r, a.y, acc.y));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {  // acc + a b
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}

// host-built tables, device copy in FmmPlan::d_tab:
//   binA[k][l] = C(l+k-1, k-1)      (k = 0..p, l = 0..p; k = 0 row unused)
//   binB[k][l] = C(k, l)            (L2L)
//   binM[k][l] = C(l-1, k-1) 2^-k   (M2M, k >= 1, l >= k)
//   dpow[c][n] = d_c^n, d_c = ((c&1) - 1/2)/2 + i((c>>1) - 1/2)/2
//   mpow[o][k] = (-1/D_o)^k, dinv[o][l] = D_o^{-l}, o = (dy+3)*7 + (dx+3)
struct FmmTabLayout {
  int p, P1;
  size_t binA, binB, binM, dpow, mpow, dinv, logd, total;  // offsets in doubles
  __host__ __device__ explicit FmmTabLayout(int p_) : p(p_), P1(p_ + 1) {
    size_t o = 0;
    binA = o; o += (size_t)P1 * P1;
    binB = o; o += (size_t)P1 * P1;
    binM = o; o += (size_t)P1 * P1;
    dpow = o; o += (size_t)4 * P1 * 2;
    mpow = o; o += (size_t)49 * P1 * 2;
    dinv = o; o += (size_t)49 * P1 * 2;
    logd = o; o += 49;
    total = o;
  }
};

inline void fmm_tables_fill(int p, std::vector<double>& t) {
  FmmTabLayout L(p);
  t.assign(L.total, 0.0);
  const int P1 = L.P1;
  // binomials in long double to keep every entry correctly rounded-ish
  auto binom = [](int n, int r) -> long double {
    if (r < 0 || r > n) return 0.0L;
    long double v = 1.0L;
    for (int i = 1; i <= r; ++i) v = v * (long double)(n - r + i) / (long double)i;
    return v;
  };
  for (int k = 0; k <= p; ++k)
    for (int l = 0; l <= p; ++l) {
      t[L.binA + (size_t)k * P1 + l] = k >= 1 ? (double)binom(l + k - 1, k - 1) : 0.0;
      t[L.binB + (size_t)k * P1 + l] = (double)binom(k, l);
      t[L.binM + (size_t)k * P1 + l] =
          (k >= 1 && l >= k) ? (double)(binom(l - 1, k - 1) * std::pow(2.0L, (long double)-k)) : 0.0;
    }
  for (int c = 0; c < 4; ++c) {
    const long double dx = ((c & 1) - 0.5L) * 0.5L, dy = ((c >> 1) - 0.5L) * 0.5L;
    long double re = 1.0L, im = 0.0L;
    for (int n = 0; n <= p; ++n) {
      t[L.dpow + ((size_t)c * P1 + n) * 2] = (double)re;
      t[L.dpow + ((size_t)c * P1 + n) * 2 + 1] = (double)im;
      const long double nr = re * dx - im * dy, ni = re * dy + im * dx;
      re = nr;
      im = ni;
    }
  }
  for (int dyi = -3; dyi <= 3; ++dyi)
    for (int dxi = -3; dxi <= 3; ++dxi) {
      const int o = (dyi + 3) * 7 + (dxi + 3);
      const long double n2 = (long double)dxi * dxi + (long double)dyi * dyi;
      if (n2 == 0.0L) continue;
      // m = -1/D = -conj(D)/|D|^2 ; Dinv = 1/D = conj(D)/|D|^2
      const long double mr = -dxi / n2, mi = dyi / n2;
      const long double ir = dxi / n2, ii = -dyi / n2;
      long double pr = 1.0L, pi = 0.0L, qr = 1.0L, qi = 0.0L;
      for (int n = 0; n <= p; ++n) {
        t[L.mpow + ((size_t)o * P1 + n) * 2] = (double)pr;
        t[L.mpow + ((size_t)o * P1 + n) * 2 + 1] = (double)pi;
        t[L.dinv + ((size_t)o * P1 + n) * 2] = (double)qr;
        t[L.dinv + ((size_t)o * P1 + n) * 2 + 1] = (double)qi;
        long double a = pr * mr - pi * mi, b = pr * mi + pi * mr;
        pr = a;
        pi = b;
        a = qr * ir - qi * ii;
        b = qr * ii + qi * ir;
        qr = a;
        qi = b;
      }
      t[L.logd + o] = (double)(0.5L * logl(n2));
    }
}

struct FmmGeom {
  double x0, y0, h0;  // root box lower-left corner and side
  int L;              // leaf level
  int p;
};

__device__ __forceinline__ int64_t lvl_off(int l) { return ((1ll << (2 * l)) - 1) / 3; }

__device__ __forceinline__ int fmm_cell(double x, double x0, double inv_h, int n) {
  const double f = floor((x - x0) * inv_h);
  return f < 0.0 ? 0 : (f >= (double)n ? n - 1 : (int)f);
}

__global__ void k_fmm_keys(int64_t S, const double* __restrict__ sx, const double* __restrict__ sy,
                           FmmGeom g, int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int n = 1 << g.L;
  const double inv_h = (double)n / g.h0;
  const int ix = fmm_cell(sx[i], g.x0, inv_h, n), iy = fmm_cell(sy[i], g.y0, inv_h, n);
  keys[i] = iy * n + ix;
  vals[i] = (int32_t)i;
}

// leaf key of every target (row-major leaf index; n*n for targets outside the
// root box), for the leaf-ordered L2P + P2P pass
__global__ void k_fmm_tkeys(int64_t T, const double2* __restrict__ txy, FmmGeom g, int32_t* __restrict__ keys,
                            int32_t* __restrict__ vals) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int n = 1 << g.L;
  const double inv_h = (double)n / g.h0;
  const double2 z = txy[t];
  const double fx = floor((z.x - g.x0) * inv_h), fy = floor((z.y - g.y0) * inv_h);
  const bool in = fx >= 0.0 && fy >= 0.0 && fx < (double)n && fy < (double)n;
  keys[t] = in ? (int)fy * n + (int)fx : n * n;
  vals[t] = (int32_t)t;
}

// Boxes whose local expansion the evaluation needs: the leaves that hold a
// target and their ancestors.  The downward pass (M2L + L2L) skips the rest,
// so a shard of the targets pays for its own part of the tree only; with
// targets in every leaf nothing is skipped.  A box's expansion does not
// depend on which other boxes are computed: u(t) stays bitwise the same.
__global__ void k_fmm_mark_leaves(int64_t T, const int32_t* __restrict__ keys, int L, uint8_t* __restrict__ active) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int64_t nleaf = 1ll << (2 * L);
  const int32_t k = keys[t];
  if ((int64_t)k < nleaf) active[lvl_off(L) + k] = 1;
}
__global__ void k_fmm_mark_parents(int l, uint8_t* __restrict__ active) {
  const int n = 1 << l;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= (int64_t)n * n) return;
  const int ix = (int)(b % n), iy = (int)(b / n);
  const uint8_t* ch = active + lvl_off(l + 1);
  const int64_t c0 = (int64_t)(2 * iy) * (2 * n) + 2 * ix;
  active[lvl_off(l) + b] = ch[c0] | ch[c0 + 1] | ch[c0 + 2 * n] | ch[c0 + 2 * n + 1];
}

__global__ void k_fmm_gather(int64_t S, const int32_t* __restrict__ idx, const double* __restrict__ sx,
                             const double* __restrict__ sy, const double* __restrict__ sq,
                             double2* __restrict__ pxy, double* __restrict__ pq) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int32_t j = idx[i];
  pxy[i] = make_double2(sx[j], sy[j]);
  pq[i] = sq[j];
}

// P2M: one warp per leaf box; lanes over the box's sources, 16 coefficients
// per round combined by fixed-order warp sums.
__global__ void __launch_bounds__(kFmmThreads)
    k_fmm_p2m(FmmGeom g, const int64_t* __restrict__ beg, const int64_t* __restrict__ end,
              const double2* __restrict__ pxy, const double* __restrict__ pq, double2* __restrict__ mp) {
  // lanes own sources while forming q w^k, then own coefficients k: the
  // 32 x P1 power table goes through shared memory and lane k sums column k
  // (fixed order), so a batch costs no warp reductions
  extern __shared__ __align__(16) unsigned char psm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n = 1 << g.L, P1 = g.p + 1;
  const int P1s = P1 | 1;  // odd row stride: the lanes' rows fall in different bank groups
  double2* tab = reinterpret_cast<double2*>(psm) + (size_t)wid * 32 * P1s;  // [source lane][k]
  const int64_t nbox = (int64_t)n * n;
  const double h = g.h0 / n;
  const int64_t base = lvl_off(g.L);
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbox;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double2* out = mp + (base + b) * P1;
    const int64_t s0 = beg[b], s1 = end[b];
    const int ix = (int)(b % n), iy = (int)(b / n);
    const double cx = g.x0 + (ix + 0.5) * h, cy = g.y0 + (iy + 0.5) * h;
    const double inv_h = 1.0 / h;
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};  // coefficients lane, lane + 32
    for (int64_t sb = s0; sb < s1; sb += 32) {
      const int64_t s = sb + lane;
      double2 w = make_double2(0.0, 0.0), pw = make_double2(0.0, 0.0);
      if (s < s1) {
        const double2 z = pxy[s];
        w = make_double2((z.x - cx) * inv_h, (z.y - cy) * inv_h);
        pw = make_double2(pq[s], 0.0);  // q w^0
      }
      __syncwarp();
      tab[lane * P1s] = pw;
      for (int k = 1; k < P1; ++k) {
        pw = cmul(pw, w);  // q w^k
        tab[lane * P1s + k] = pw;
      }
      __syncwarp();
      const int nb = (int)min((int64_t)32, s1 - sb);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = lane + 32 * r;
        if (k >= P1) continue;
        double2 a = acc[r];
        for (int j = 0; j < nb; ++j) {
          const double2 v = tab[j * P1s + k];
          a.x += v.x;
          a.y += v.y;
        }
        acc[r] = a;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int k = lane + 32 * r;
      if (k >= P1) continue;
      out[k] = k == 0 ? make_double2(acc[r].x, 0.0) : make_double2(-acc[r].x / k, -acc[r].y / k);
    }
  }
}

// M2M: one warp per parent box at level l (children at level l+1)
__global__ void __launch_bounds__(kFmmThreads)
    k_fmm_m2m(FmmGeom g, int l, const double* __restrict__ tab, double2* __restrict__ mp) {
  extern __shared__ double fsh[];
  FmmTabLayout TL(g.p);
  const int P1 = TL.P1;
  const int P1e = (P1 * P1 + 1) & ~1;               // keep double2 16-B aligned
  double* binM = fsh;                              // P1*P1
  double2* dpow = (double2*)(fsh + P1e);           // 4*P1
  for (int i = threadIdx.x; i < P1 * P1; i += blockDim.x) binM[i] = tab[TL.binM + i];
  for (int i = threadIdx.x; i < 4 * P1; i += blockDim.x)
    dpow[i] = make_double2(tab[TL.dpow + 2 * i], tab[TL.dpow + 2 * i + 1]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int n = 1 << l;
  const int64_t nbox = (int64_t)n * n;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbox;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int ix = (int)(b % n), iy = (int)(b / n);
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    double Q = 0.0;
    for (int c = 0; c < 4; ++c) {
      const int cx = 2 * ix + (c & 1), cy = 2 * iy + (c >> 1);
      const double2* ch = mp + (lvl_off(l + 1) + (int64_t)cy * (2 * n) + cx) * P1;
      const double Qc = ch[0].x;
      Q += Qc;
      if (Qc == 0.0) {
        bool any = false;
        for (int k = lane; k < P1; k += 32) any |= (ch[k].x != 0.0 || ch[k].y != 0.0);
        if (!__any_sync(0xffffffffu, any)) continue;
      }
      const double2* dp = dpow + c * P1;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int ll = lane + 32 * r;
        if (ll < 1 || ll >= P1) continue;
        double2 s = make_double2(-Qc * dp[ll].x / ll, -Qc * dp[ll].y / ll);
        for (int k = 1; k <= ll; ++k) s = cfma(ch[k], make_double2(binM[k * P1 + ll] * dp[ll - k].x,
                                                                  binM[k * P1 + ll] * dp[ll - k].y), s);
        acc[r].x += s.x;
        acc[r].y += s.y;
      }
    }
    double2* out = mp + (lvl_off(l) + b) * P1;
    if (lane == 0) out[0] = make_double2(Q, 0.0);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int ll = lane + 32 * r;
      if (ll >= 1 && ll < P1) out[ll] = acc[r];
    }
  }
}

// Downward pass at level l: local(B) = L2L(local(parent)) + sum_{C in IL(B)} M2L(C -> B).
// One warp per box; lanes own coefficients l = lane, lane + 32.
__global__ void __launch_bounds__(kFmmThreads)
    k_fmm_m2l(FmmGeom g, int l, const double* __restrict__ tab, const double2* __restrict__ mp,
              double2* __restrict__ lp, const uint8_t* __restrict__ active) {
  extern __shared__ double fsh[];
  FmmTabLayout TL(g.p);
  const int P1 = TL.P1;
  const int P1e = (P1 * P1 + 1) & ~1;                // keep double2 16-B aligned
  double* binA = fsh;                               // [k][l]
  double* binB = binA + P1e;                        // [k][l]
  double2* dpow = (double2*)(binB + P1e);           // [4][P1]
  double2* ebuf = dpow + 4 * P1;                    // per warp [P1]
  for (int i = threadIdx.x; i < P1 * P1; i += blockDim.x) {
    binA[i] = tab[TL.binA + i];
    binB[i] = tab[TL.binB + i];
  }
  for (int i = threadIdx.x; i < 4 * P1; i += blockDim.x)
    dpow[i] = make_double2(tab[TL.dpow + 2 * i], tab[TL.dpow + 2 * i + 1]);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double2* e = ebuf + wid * P1;
  const int n = 1 << l;
  const int64_t nbox = (int64_t)n * n;
  const double h = g.h0 / n;
  const double logh = log(h);
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbox;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (!active[lvl_off(l) + b]) continue;  // no target below this box
    const int ix = (int)(b % n), iy = (int)(b / n);
    double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    if (l >= 3) {  // L2L from the parent (levels 0-2 carry no local expansion)
      const int px = ix >> 1, py = iy >> 1, c = (ix & 1) | ((iy & 1) << 1);
      const double2* par = lp + (lvl_off(l - 1) + (int64_t)py * (n >> 1) + px) * P1;
      const double2* dp = dpow + c * P1;
      __syncwarp();
      for (int k = lane; k < P1; k += 32) e[k] = par[k];
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int ll = lane + 32 * r;
        if (ll >= P1) continue;
        double2 s = make_double2(0.0, 0.0);
        for (int k = ll; k < P1; ++k) {
          const double bb = binB[k * P1 + ll];
          s = cfma(e[k], make_double2(bb * dp[k - ll].x, bb * dp[k - ll].y), s);
        }
        const double sc = ldexp(1.0, -ll);
        acc[r] = make_double2(s.x * sc, s.y * sc);
      }
    }
    // interaction list: children of the parent's neighbours not adjacent to B
    const int px = ix >> 1, py = iy >> 1;
    for (int cy = 2 * py - 2; cy <= 2 * py + 3; ++cy) {
      if (cy < 0 || cy >= n) continue;
      for (int cx = 2 * px - 2; cx <= 2 * px + 3; ++cx) {
        if (cx < 0 || cx >= n) continue;
        const int dxi = cx - ix, dyi = cy - iy;
        if (dxi >= -1 && dxi <= 1 && dyi >= -1 && dyi <= 1) continue;
        const double2* src = mp + (lvl_off(l) + (int64_t)cy * n + cx) * P1;
        const double Q = src[0].x;
        const int o = (dyi + 3) * 7 + (dxi + 3);
        const double* mpw = tab + TL.mpow + (size_t)o * P1 * 2;
        const double* dnv = tab + TL.dinv + (size_t)o * P1 * 2;
        // e_k = a_k (-1/D)^k  (k >= 1), e_0 = 0
        bool any = Q != 0.0;
        __syncwarp();
        for (int k = lane; k < P1; k += 32) {
          const double2 a = src[k];
          any |= (k >= 1) && (a.x != 0.0 || a.y != 0.0);
          e[k] = k == 0 ? make_double2(0.0, 0.0) : cmul(a, make_double2(mpw[2 * k], mpw[2 * k + 1]));
        }
        if (!__any_sync(0xffffffffu, any)) continue;  // empty source box
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int ll = lane + 32 * r;
          if (ll >= P1) continue;
          double2 s = make_double2(0.0, 0.0);
          for (int k = 1; k < P1; ++k) s = cfma_r(binA[k * P1 + ll], e[k], s);
          if (ll == 0) {
            acc[r].x += s.x + Q * (logh + tab[TL.logd + o]);
            acc[r].y += s.y;
          } else {
            s.x -= Q / ll;
            acc[r] = cfma(s, make_double2(dnv[2 * ll], dnv[2 * ll + 1]), acc[r]);
          }
        }
      }
    }
    double2* out = lp + (lvl_off(l) + b) * P1;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int ll = lane + 32 * r;
      if (ll < P1) out[ll] = acc[r];
    }
  }
}

// The same downward pass specialised to P1 = p + 1 <= 32 coefficients, one per
// lane: lane l keeps its column binA[1..p][l] of the M2L binomial matrix in
// registers, so each source box costs p broadcast loads of e_k and 2 p DFMA
// per lane instead of two shared loads per pair of DFMA.  Instantiated for
// the orders vp_fmm_order_for returns (P1 = 8, 12, .., 32; lanes >= P1 idle).
template <int P1>
__global__ void __launch_bounds__(kFmmThreads)
    k_fmm_m2l32(FmmGeom g, int l, const double* __restrict__ tab, const double2* __restrict__ mp,
                double2* __restrict__ lp, const uint8_t* __restrict__ active) {
  static_assert(P1 >= 2 && P1 <= 32, "one coefficient per lane");
  __shared__ double binB[P1 * P1];
  __shared__ double2 dpow[4 * P1];
  __shared__ double2 ebuf[kFmmThreads / 32][P1];
  FmmTabLayout TL(P1 - 1);
  for (int i = threadIdx.x; i < P1 * P1; i += blockDim.x) binB[i] = tab[TL.binB + i];
  for (int i = threadIdx.x; i < 4 * P1; i += blockDim.x)
    dpow[i] = make_double2(tab[TL.dpow + 2 * i], tab[TL.dpow + 2 * i + 1]);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double bc[P1];
#pragma unroll
  for (int k = 1; k < P1; ++k) bc[k] = lane < P1 ? tab[TL.binA + k * P1 + lane] : 0.0;
  __syncthreads();
  double2* e = ebuf[wid];
  const double inv_l = lane > 0 ? 1.0 / lane : 0.0;
  const double scl = ldexp(1.0, -lane);
  const int n = 1 << l;
  const int64_t nbox = (int64_t)n * n;
  const double h = g.h0 / n;
  const double logh = log(h);
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nbox;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (!active[lvl_off(l) + b]) continue;  // no target below this box
    const int ix = (int)(b % n), iy = (int)(b / n);
    double2 acc = make_double2(0.0, 0.0);
    if (l >= 3) {  // L2L from the parent (levels 0-2 carry no local expansion)
      const int px = ix >> 1, py = iy >> 1, c = (ix & 1) | ((iy & 1) << 1);
      const double2* par = lp + (lvl_off(l - 1) + (int64_t)py * (n >> 1) + px) * P1;
      const double2* dp = dpow + c * P1;
      __syncwarp();
      if (lane < P1) e[lane] = par[lane];
      __syncwarp();
      double2 s = make_double2(0.0, 0.0);
      for (int k = lane; k < P1; ++k) {
        const double bb = binB[k * P1 + lane];
        s = cfma(e[k], make_double2(bb * dp[k - lane].x, bb * dp[k - lane].y), s);
      }
      acc = make_double2(s.x * scl, s.y * scl);
    }
    // interaction list: children of the parent's neighbours not adjacent to B
    const int px = ix >> 1, py = iy >> 1;
    for (int cy = 2 * py - 2; cy <= 2 * py + 3; ++cy) {
      if (cy < 0 || cy >= n) continue;
      for (int cx = 2 * px - 2; cx <= 2 * px + 3; ++cx) {
        if (cx < 0 || cx >= n) continue;
        const int dxi = cx - ix, dyi = cy - iy;
        if (dxi >= -1 && dxi <= 1 && dyi >= -1 && dyi <= 1) continue;
        const double2* src = mp + (lvl_off(l) + (int64_t)cy * n + cx) * P1;
        const double2 a = lane < P1 ? src[lane] : make_double2(0.0, 0.0);
        const double Q = __shfl_sync(0xffffffffu, a.x, 0);
        const int o = (dyi + 3) * 7 + (dxi + 3);
        const double* mpw = tab + TL.mpow + (size_t)o * P1 * 2;
        const double* dnv = tab + TL.dinv + (size_t)o * P1 * 2;
        // e_k = a_k (-1/D)^k  (k >= 1), e_0 = 0
        const bool any = Q != 0.0 || (lane >= 1 && (a.x != 0.0 || a.y != 0.0));
        if (!__any_sync(0xffffffffu, any)) continue;  // empty source box
        __syncwarp();
        if (lane < P1)
          e[lane] = lane == 0 ? make_double2(0.0, 0.0) : cmul(a, make_double2(mpw[2 * lane], mpw[2 * lane + 1]));
        __syncwarp();
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 1; k < P1; ++k) s = cfma_r(bc[k], e[k], s);
        if (lane == 0) {
          acc.x += s.x + Q * (logh + tab[TL.logd + o]);
          acc.y += s.y;
        } else if (lane < P1) {
          s.x -= Q * inv_l;
          acc = cfma(s, make_double2(dnv[2 * lane], dnv[2 * lane + 1]), acc);
        }
      }
    }
    if (lane < P1) lp[(lvl_off(l) + b) * P1 + lane] = acc;
  }
}

// L2P + P2P: one thread per target inside the root box.  Targets outside
// are flagged (flag[t] = 1) and summed by the direct kernel.
template <bool ZERO_CHECK>
__global__ void __launch_bounds__(256)
    k_fmm_eval(int64_t T, const double2* __restrict__ txy, FmmGeom g, const int64_t* __restrict__ beg,
               const int64_t* __restrict__ end, const double2* __restrict__ pxy,
               const double* __restrict__ pq, const double2* __restrict__ lp, double* __restrict__ u,
               int32_t* __restrict__ flag, unsigned c3ff, const int32_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char fsm[];
  double2* ltab = reinterpret_cast<double2*>(fsm);
  for (int i = threadIdx.x; i < kLogEntries * kLogCopies; i += blockDim.x) ltab[i] = g_logtab[i / kLogCopies];
  __syncthreads();
  const unsigned laneoff = 16u * (threadIdx.x & (kLogCopies - 1));
  // targets in leaf order (`order`, a stable sort by leaf key): a warp's
  // threads share their leaf, so the expansion and source loads broadcast
  const int64_t ti = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (ti >= T) return;
  const int64_t t = order ? (int64_t)order[ti] : ti;
  const double2 z = txy[t];
  const int n = 1 << g.L, P1 = g.p + 1;
  const double inv_h = (double)n / g.h0, h = g.h0 / n;
  const double fx = floor((z.x - g.x0) * inv_h), fy = floor((z.y - g.y0) * inv_h);
  if (!(fx >= 0.0 && fy >= 0.0 && fx < (double)n && fy < (double)n)) {
    flag[t] = 1;
    u[t] = 0.0;
    return;
  }
  flag[t] = 0;
  const int ix = (int)fx, iy = (int)fy;
  // L2P (Horner in eta)
  const double2* loc = lp + (lvl_off(g.L) + (int64_t)iy * n + ix) * P1;
  const double2 eta = make_double2((z.x - (g.x0 + (ix + 0.5) * h)) / h, (z.y - (g.y0 + (iy + 0.5) * h)) / h);
  double2 phi = loc[P1 - 1];
  for (int k = P1 - 2; k >= 0; --k) phi = cfma(phi, eta, loc[k]);
  double acc = 2.0 * phi.x;
  // P2P over the 3x3 neighbour leaves
  double sacc = 0.0;
  for (int cy = iy - 1; cy <= iy + 1; ++cy) {
    if (cy < 0 || cy >= n) continue;
    for (int cx = ix - 1; cx <= ix + 1; ++cx) {
      if (cx < 0 || cx >= n) continue;
      const int64_t c = (int64_t)cy * n + cx;
      const int64_t s1 = end[c];
      int64_t s = beg[c];
      // four sources per step: their loads issue together (latency-bound otherwise)
      for (; s + 4 <= s1; s += 4) {
        double2 ps[4];
        double q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ps[i] = pxy[s + i];
          q[i] = pq[s + i];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double dx = z.x - ps[i].x, dy = z.y - ps[i].y;
          sacc = fma(q[i], far_log_r2<ZERO_CHECK>(ltab, laneoff, c3ff, fma(dx, dx, dy * dy)), sacc);
        }
      }
      for (; s < s1; ++s) {
        const double2 ps = pxy[s];
        const double dx = z.x - ps.x, dy = z.y - ps.y;
        sacc = fma(pq[s], far_log_r2<ZERO_CHECK>(ltab, laneoff, c3ff, fma(dx, dx, dy * dy)), sacc);
      }
    }
  }
  u[t] = acc + sacc;
}

// gather / scatter for the targets outside the root box (direct far sum)
__global__ void k_gather_targets(int64_t n, const int32_t* __restrict__ idx, const double2* __restrict__ txy,
                                 double2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = txy[idx[i]];
}
__global__ void k_scatter_add(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ v,
                              double* __restrict__ u) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[idx[i]] = v[i];
}
