// koorn.cuh -- orthonormal Koornwinder basis on the reference simplex,
// shared by host setup (vp_setup.cpp) and device kernels (vp_kernels.cu).
//
// Basis definition and index order follow the reference:
//   K_mn(x,y) = c_mn P_{n-m}^{(2m+1,0)}(2x-1) (1-x)^m P_m(2y/(1-x)-1),
//   c_mn = sqrt((2m+1)(2n+2)), index n(n+1)/2 + m   (koornwinder.hpp:12-21)
// evaluated by a homogenised Legendre recurrence in (u, v) = (2y-(1-x), 1-x)
// and the Jacobi P^{(2m+1,0)} three-term recurrence (koornwinder.hpp:77-113).
// The device path uses host-precomputed recurrence coefficients (no
// divisions) and fuses the contraction with the density coefficients.
#pragma once
#include <cmath>

#ifdef __CUDACC__
#define VP_HD __host__ __device__ __forceinline__
#else
#define VP_HD inline
#endif

namespace vp {

VP_HD constexpr int koorn_size(int p) { return (p + 1) * (p + 2) / 2; }
VP_HD constexpr int koorn_index(int m, int n) { return n * (n + 1) / 2 + m; }

constexpr int kMaxP = 12;

// All K_mn, m+n <= N, at (x, y).
VP_HD void koorn_eval(int N, double x, double y, double* out) {
  double L[kMaxP + 2];
  const double v = 1.0 - x;
  const double u = 2.0 * y - v;
  const double v2 = v * v;
  L[0] = 1.0;
  if (N >= 1) L[1] = u;
  for (int m = 1; m + 1 <= N; ++m)
    L[m + 1] = ((2 * m + 1) * (u * L[m]) - double(m) * (v2 * L[m - 1])) / double(m + 1);
  const double t = 2.0 * x - 1.0;
  for (int m = 0; m <= N; ++m) {
    const double a = 2 * m + 1;
    double p0 = 1.0, p1 = 0.5 * (a + (a + 2.0) * t);
    for (int k = 0; m + k <= N; ++k) {
      const int n = m + k;
      const double pk = (k == 0) ? p0 : p1;
      out[koorn_index(m, n)] = sqrt((double)((2 * m + 1) * (2 * n + 2))) * (pk * L[m]);
      if (k >= 1 && m + k + 1 <= N) {
        const double kk = k;
        const double c1 = 2 * (kk + 1) * (kk + a + 1) * (2 * kk + a);
        const double c2 = (2 * kk + a + 1) * (a * a);
        const double c3 = (2 * kk + a) * (2 * kk + a + 1) * (2 * kk + a + 2);
        const double c4 = 2 * (kk + a) * kk * (2 * kk + a + 2);
        const double p2 = ((c2 * p1 + c3 * (t * p1)) - c4 * p0) / c1;
        p0 = p1;
        p1 = p2;
      }
    }
  }
}

// Division-free recurrence table for the device path.  For the Legendre
// part: L_{m+1} = la[m] u L_m - lb[m] v^2 L_{m-1}.  For each m the Jacobi
// P^{(2m+1,0)}_{k+1} = (ja t + jb) P_k - jc P_{k-1}, P_1 = j1a t + j1b, and
// the normalisation c_mn.  Laid out for p <= kMaxP.
struct KoornTable {
  double la[kMaxP + 1], lb[kMaxP + 1];
  double j1a[kMaxP + 1], j1b[kMaxP + 1];
  // per (m, k) with k >= 1: index m*(kMaxP+1)+k
  double ja[(kMaxP + 1) * (kMaxP + 1)], jb[(kMaxP + 1) * (kMaxP + 1)],
      jc[(kMaxP + 1) * (kMaxP + 1)];
  double cn[(kMaxP + 1) * (kMaxP + 2) / 2];
};

inline void koorn_table_fill(KoornTable& T) {
  for (int m = 0; m <= kMaxP; ++m) {
    T.la[m] = m >= 1 ? double(2 * m + 1) / double(m + 1) : 1.0;
    T.lb[m] = m >= 1 ? double(m) / double(m + 1) : 0.0;
    const double a = 2 * m + 1;
    T.j1a[m] = 0.5 * (a + 2.0);
    T.j1b[m] = 0.5 * a;
    for (int k = 0; k <= kMaxP; ++k) {
      const int i = m * (kMaxP + 1) + k;
      if (k == 0) {
        T.ja[i] = T.jb[i] = T.jc[i] = 0.0;
        continue;
      }
      const double kk = k;
      const double c1 = 2 * (kk + 1) * (kk + a + 1) * (2 * kk + a);
      const double c2 = (2 * kk + a + 1) * (a * a);
      const double c3 = (2 * kk + a) * (2 * kk + a + 1) * (2 * kk + a + 2);
      const double c4 = 2 * (kk + a) * kk * (2 * kk + a + 2);
      T.ja[i] = c3 / c1;
      T.jb[i] = c2 / c1;
      T.jc[i] = c4 / c1;
    }
  }
  for (int n = 0; n <= kMaxP; ++n)
    for (int m = 0; m <= n; ++m) T.cn[koorn_index(m, n)] = std::sqrt((double)((2 * m + 1) * (2 * n + 2)));
}

}  // namespace vp
