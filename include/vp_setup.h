/* vp_setup.h -- host-side setup for the volume-potential evaluator.
 *
 * Everything here runs once per problem on the host (C++), producing the
 * inputs the evaluator's C-ABI (vp.h) consumes: quadrature rules on the
 * reference simplex, the 1-D rules of self-interaction, synthetic meshes,
 * target sets and per-triangle Koornwinder density coefficients.
 *
 * Reference anchors:
 *   - rules are data in the reference (rules.hpp:88-125); its
 *     Xiao-Gimbutas / Vioreanu-Rokhlin tables are absent, so
 *     vps_quad_rule gives the evaluation's far / near rules -- fully symmetric
 *     rules from this repository's own moment-fitting solver for orders 6, 10
 *     and 12, vps_simplex_rule's collapsed Gauss-Jacobi rule otherwise -- all
 *     passing the reference's validate_rule contract (rules.hpp:60-85);
 *   - vps_gauss_legendre restates gauss_legendre (gauss.hpp:17-46);
 *   - vps_ggq restates build_ggq's moment fitting (ggq.hpp:33-182);
 *   - density coefficients replace the reference's callable f
 *     with per-triangle order-p Koornwinder coefficients (BASELINE.json north_star).
 * Return codes: 0 ok, 1 usage error, 2 numerical failure.
 */
#ifndef VP_SETUP_H
#define VP_SETUP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* number of Koornwinder modes (p+1)(p+2)/2 (koornwinder.hpp:20) */
int vps_koorn_size(int p);

/* Gauss-Legendre on [-1,1] (gauss.hpp:17-46) */
int vps_gauss_legendre(int n, double* x, double* w);

/* Gauss-Jacobi for the weight (1-u) on [0,1], n nodes */
int vps_gauss_jacobi10(int n, double* x, double* w);

/* Simplex rule exact to total degree `order`: collapsed Gauss-Jacobi with
 * n = floor(order/2)+1 points per direction, len = n*n.  Query the length
 * with x == NULL. */
int vps_simplex_rule(int order, int* len, double* x, double* y, double* w);
/* The evaluation's far / near rule of order `order` (load_far_rule, rules.hpp:
 * 121-125): a fully symmetric rule with positive weights and interior points,
 * exact to degree `order`, computed by this repository's own moment-fitting
 * solver (tools/make_sym_rules.py; degrees 6, 10 and 12: 12, 25 and 33
 * points), else vps_simplex_rule's collapsed Gauss-Jacobi rule.  Same calling
 * convention (x == NULL: only *len). */
int vps_quad_rule(int order, int* len, double* x, double* y, double* w);

/* Radial generalized Gaussian rule: ng+1 nodes on (0,1) integrating
 * r P_n(2r-1) and r log r P_n(2r-1), n <= ng (ggq.hpp:13-22, :96-182). */
int vps_ggq(int ng, double* r, double* w, double* max_residual);

/* Circular arc gamma(tau L), tau in [0,1], as a Legendre series of degree
 * deg (coefficients of P_n(2 tau - 1)); *len = arc length.  Curved-element
 * input of vp_set_curves. */
int vps_circle_arc(double cx, double cy, double R, double th0, double th1, int deg, double* gx, double* gy,
                   double* len);

/* Closed boundary curves with arc-length parametrisation (the reference's
 * curve layer, curve.hpp:16-332: ParamCurve kinds + ArcLengthCurve), used to
 * build the per-element Legendre series of vp_set_curves (SPEC.md:200-210
 * annotate_boundary).  Parameter t in [0, 1]; arc length s in [0, L). */
typedef struct vps_curve vps_curve;
enum {
  VPS_CURVE_CIRCLE = 0,  /* (cx, cy, r): c + r (cos 2 pi t, sin 2 pi t)        curve.hpp:25-45 */
  VPS_CURVE_ELLIPSE = 1, /* (a, b): (a cos 2 pi t, b sin 2 pi t)                curve.hpp:47-67 */
  VPS_CURVE_WOBBLY = 2,  /* (a, b, k): polar r = a + b cos(k theta), a > |b|    curve.hpp:69-101 */
  VPS_CURVE_HERMITE = 3, /* n x (t, x, y, dx, dy): periodic cubic Hermite       curve.hpp:103-162 */
  VPS_CURVE_ARC = 4      /* (cx, cy, r, th0, th1): closed only if |th1-th0| = 2 pi */
};
/* Errors: 1 with "reparametrize: curve is not closed" when |gamma(0) -
 * gamma(1)| > 1e-8 L (curve.hpp:250-252); Hermite parameter checks as
 * curve.hpp:108-116. */
int vps_curve_create(int kind, const double* params, int n_params, vps_curve** out);
void vps_curve_destroy(vps_curve* c);
double vps_curve_length(const vps_curve* c);
int vps_curve_ccw(const vps_curve* c);
/* s -> t (the arc-length inverse) */
int vps_curve_param(const vps_curve* c, double s, double* t);
/* Gamma(s), unit tangent Gamma'(s) and Gamma''(s) at n arc lengths (s wraps
 * modulo L); tangent/dd may be NULL */
int vps_curve_points(const vps_curve* c, int64_t n, const double* s, double* xy, double* tangent, double* dd);
/* closest point: s and distance for n points (sdf.hpp:56-80 closest_point) */
int vps_curve_closest(const vps_curve* c, int64_t n, const double* xy, double* s, double* dist);
/* G(tau) = Gamma(s_from + tau (s_to - s_from)), tau in [0,1], as a degree-deg
 * Legendre series in P_n(2 tau - 1); *len = |s_to - s_from| */
int vps_curve_segment(const vps_curve* c, double s_from, double s_to, int deg, double* gx, double* gy,
                      double* len);
const char* vps_curve_last_error(void);

/* Target nodes on the reference simplex: shifted principal lattice
 * ((i+1)/(p+3), (j+1)/(p+3)), i+j <= p; (p+1)(p+2)/2 nodes. */
int vps_lattice_nodes(int p, double* x, double* y);

/* analytic densities used by the synthetic configurations */
enum {
  VPS_F_CONST = 0,     /* params[0] */
  VPS_F_SQUARE = 1,    /* sin(3x)cos(2y) + x^2 */
  VPS_F_GAUSS = 2,     /* exp(-params[2] |x-(params[0],params[1])|^2) */
  VPS_F_BUMPS = 3,     /* sum_k A_k exp(-|x-c_k|^2/s_k^2), params = n_bumps x (cx,cy,s,A) */
  VPS_F_COSSIN = 4,    /* cos(4 pi x) sin(2 pi y) */
  VPS_F_LINEAR = 5     /* params[0] + params[1] x + params[2] y */
};
double vps_density_eval(int kind, const double* params, int n_params, double x, double y);

/* L2 projection of an analytic density onto the order-p Koornwinder basis
 * of every triangle: c_T,j = int_{Delta^1} f(rho_T(xi)) K_j(xi) dxi. */
int vps_project_density(int64_t n_vert, const double* vxy, int64_t n_tri, const int32_t* tri,
                        int p, int kind, const double* params, int n_params, double* coeffs);

/* Synthetic configurations of BASELINE.json:configs (1-based id 1..5).
 * q_override > 0 replaces the config's far order (config 5 sweep). */
typedef struct {
  int64_t n_vert;
  int64_t n_tri;
  int64_t n_tgt;
  int p;
  int q;
  int density_kind;
  int n_params;
  double params[64];
  double eps;
  uint64_t seed;
  int staggered; /* targets on a separate staggered mesh */
  int pad;
} vps_config_info;

int vps_config_info_get(int config, int q_override, uint64_t seed, vps_config_info* info);
int vps_config_fill(int config, int q_override, uint64_t seed, double* vxy, int32_t* tri,
                    double* txy, double* coeffs);

const char* vps_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
