/* vp_oracle.h -- CPU oracle for the volume-potential hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is a plain C++ restatement of the
 * reference's specified algorithm and
 * of the reference's implemented foundations (koornwinder.hpp, rules.hpp,
 * gauss.hpp, quadtree.hpp).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it, and only as
 * the checker.  The product path (libvp_b200.so) never links or calls it.
 *
 * Parity status: the hot path itself does not exist in the reference
 * (SURVEY.md §0.1), so hot-path results are "parity unpinned" against the
 * reference; the foundations this oracle is built from (Koornwinder basis,
 * Gauss-Legendre, quadtree queries, the GGQ table) are pinned against the
 * reference headers compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile) and against golden fixtures in tests/golden/.
 */
#ifndef VP_ORACLE_H
#define VP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n_vert;
  const double* vxy; /* [n_vert*2] */
  int64_t n_tri;
  const int32_t* tri; /* [n_tri*3], counter-clockwise */
  int p;
  const double* coeffs; /* [n_tri * (p+1)(p+2)/2], graded Koornwinder order */
  int q;                /* far rule order */
  int len_q;
  const double* far_x;
  const double* far_y;
  const double* far_w;
  int n_n; /* near rule order (12) */
  int len_n;
  const double* near_x;
  const double* near_y;
  const double* near_w;
  int n_l; /* Gauss-Legendre length for the arc-length direction */
  const double* gl_x; /* on [-1,1] */
  const double* gl_w;
  int n_g; /* GGQ order; n_g+1 nodes */
  const double* ggq_r;
  const double* ggq_w;
  double eps;
  int near_model;      /* 0 precise (Bernstein ellipses), 1 ball */
  int pad_;
  double ball_factor;  /* ball = circumscribed circle scaled by this (1.5) */
  /* curved (blending-map) elements: curve_id[e] >= 0 marks
   * element e as curved with vertex order (gamma(L), gamma(0), O) and its
   * side gamma(tau L) = sum_n c_n P_n(2 tau - 1), tau in [0,1]; NULL = all straight */
  const int32_t* curve_id;
  int curve_deg;
  int pad2_;
  const double* curve_cx; /* [n_curves * (curve_deg+1)] */
  const double* curve_cy;
  const double* curve_len;
} vpo_problem;

typedef struct {
  int64_t n_targets;
  int64_t n_outside;    /* targets with S(t) = -1 */
  int64_t n_near_pairs; /* sum |N(t)| */
  int64_t n_self;       /* targets with a self pair */
  int64_t n_leaves;     /* accepted near sub-simplices (s_n numerator) */
  int64_t n_panels;     /* arc-length panels (s_l numerator) */
  int64_t n_rho_le1;    /* sub-simplices accepted because rho_d <= 1 */
  int64_t n_degenerate; /* self sub-triangles skipped (h <= 1e-13 L) */
  int32_t max_depth;
  int32_t pad;
} vpo_stats;

/* foundations */
int vpo_koornwinder(int order, double x, double y, double* out);
double vpo_cn_lookup(int n);
double vpo_w_edge(int len, const double* x, const double* y, const double* w);
int vpo_validate_rule(int order, int len, const double* x, const double* y, const double* w);
int vpo_gauss_legendre(int n, double* x, double* w);
int vpo_quadtree_query(int64_t n_pts, const double* pts, int leaf_cap, double lox, double loy,
                       double hix, double hiy, int32_t* out, int64_t cap, int64_t* n_out,
                       int64_t* visited);

/* hot path */
int vpo_element_models(const vpo_problem* pr, double* rho0, double* rho0n, double* two_a);
int vpo_nearlist(const vpo_problem* pr, int64_t n_tgt, const double* txy, int32_t* self_out,
                 int64_t* offsets, int32_t* ids, int64_t ids_cap, int64_t* n_ids);
int vpo_sources(const vpo_problem* pr, double* sx, double* sy, double* q);
int vpo_far_sum(const vpo_problem* pr, int64_t n_tgt, const double* txy, int nthreads,
                double* u_far);
int vpo_near_pair(const vpo_problem* pr, double tx, double ty, int32_t elem, double* val,
                  double* sub, int64_t* leaves, int32_t* depth);
int vpo_self(const vpo_problem* pr, double tx, double ty, int32_t elem, double* val,
             double* sub, int64_t* panels);
int vpo_evaluate(const vpo_problem* pr, int64_t n_tgt, const double* txy, int nthreads,
                 double* u, double* u_far, vpo_stats* st);
const char* vpo_last_error(void);

/* Persistent oracle context: Setup::init once (element models, quadtree,
 * sources), then any number of evaluations over target batches.  The
 * problem's arrays must outlive the context. */
typedef struct vpo_ctx vpo_ctx;
int vpo_open(const vpo_problem* pr, vpo_ctx** out);
int vpo_ctx_evaluate(vpo_ctx* ctx, int64_t n_tgt, const double* txy, int nthreads, double* u,
                     double* u_far, vpo_stats* st);
void vpo_close(vpo_ctx* ctx);

/* ---- the oracle's own inputs (vp_oracle_inputs.cpp) ------------------- */
typedef struct {
  int64_t n_vert;
  int64_t n_tri;
  int64_t n_tgt;
  int p;
  int q;
  int density_kind; /* 0 const, 1 sin3x cos2y + x^2, 2 gauss, 3 bumps, 4 cos4pix sin2piy, 5 linear */
  int n_params;
  double params[64];
  double eps;
  uint64_t seed;
  int staggered;
  int pad;
} vpo_config_info;

int vpo_lattice_nodes(int p, double* x, double* y);
int vpo_gauss_jacobi10(int n, double* x, double* w);
int vpo_simplex_rule(int order, int* len, double* x, double* y, double* w);
int vpo_quad_rule(int order, int* len, double* x, double* y, double* w);
int vpo_ggq(int ng, double* r, double* w, double* max_residual);
double vpo_density_eval(int kind, const double* params, int n_params, double x, double y);
int vpo_project_density(int64_t n_vert, const double* vxy, int64_t n_tri, const int32_t* tri, int p,
                        int kind, const double* params, int n_params, double* coeffs);
int vpo_config_info_get(int config, int q_override, uint64_t seed, vpo_config_info* info);
int vpo_config_fill(int config, int q_override, uint64_t seed, double* vxy, int32_t* tri, double* txy,
                    double* coeffs);
const char* vpo_inputs_last_error(void);

/* ---- acceptance checks (vp_oracle_accept.cpp) ------------------------- */
/* Adaptive I_T(x) = int_T log|x-y| f(y) dA at points outside the triangle
 * tri = (ax, ay, bx, by, cx, cy); fkind 0: 1, 1: sin(x+2y), 2: exp(-x^2-y^2),
 * 3: Koornwinder expansion of order p in T's reference coordinates. */
int vpo_adaptive_log_integral(const double* tri, int fkind, int p, const double* coeffs, int64_t n,
                              const double* pts, double tol, int nthreads, double* out);

#ifdef __cplusplus
}
#endif
#endif
