/* vp.h -- C-ABI of the B200 volume-potential evaluator (libvp_b200.so).
 *
 * Drop-in for the hot path of the reference's evaluate_field
 * (SPEC.md:582-590): mesh + per-triangle order-p Koornwinder density in,
 * potentials u(x) = (1/2pi) int log|x-y| f(y) dy at targets out.  The
 * reference has no FFI layer of its own; each entry point
 * cites the reference (SPEC) operation it replaces.  INTEGRATION.md shows
 * the binding a reference maintainer would add.
 *
 * Conventions (mirroring the reference):
 *   - plain pointers and sizes, caller owns every host array;
 *   - a context is bound to one CUDA device (one process per GPU) and is
 *     immutable between vp_set_* calls; vp_evaluate on one context is
 *     serialised on its stream, distinct contexts may run concurrently
 *     (SPEC.md:543, :623-624);
 *   - return 0 ok, 1 usage / invalid argument, 2 numerical failure,
 *     3 device error (SPEC.md:730 exit codes + a device code); the message
 *     names the violated invariant (rules.hpp:58-85) via vp_last_error.
 *   - there is no CPU fallback: without a usable sm_100 device every
 *     compute entry point returns 3.
 */
#ifndef VP_H
#define VP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vp_ctx vp_ctx;

/* Rules on the reference simplex Delta^1 = {x,y >= 0, x+y <= 1}.
 * Replaces load_far_rule / load_rule (rules.hpp:88-125), the near rule of
 * near_eval (N_n) and the SelfRule:
 * radial GGQ (ggq.hpp:17-22) and Gauss-Legendre (gauss.hpp:17-46). */
typedef struct {
  int q;          /* far rule polynomial order N (sizes the near field) */
  int len_q;
  const double* far_x;
  const double* far_y;
  const double* far_w;
  int n_n;        /* near rule order N_n (12) */
  int len_n;
  const double* near_x;
  const double* near_y;
  const double* near_w;
  int n_l;        /* Gauss-Legendre length N_l (16), nodes on [-1,1] */
  const double* gl_x;
  const double* gl_w;
  int n_g;        /* GGQ order N_g (8): n_g+1 nodes on (0,1) */
  const double* ggq_r;
  const double* ggq_w;
  double eps;     /* tolerance epsilon of the near-field model (for:rho0) */
} vp_rules;

typedef struct {
  int64_t n_targets;
  int64_t n_outside;    /* targets with S(t) = -1 (exclusion list) */
  int64_t n_near_pairs; /* sum |N(t)| */
  int64_t n_self;       /* targets with a self pair */
  int64_t n_leaves;     /* accepted near sub-simplices; s_n = n_leaves / n_targets */
  int64_t n_panels;     /* arc-length panels; s_l = n_panels / n_self */
  int64_t n_rho_le1;    /* sub-simplices accepted with rho_d <= 1 */
  int64_t n_degenerate; /* self sub-triangles skipped (target on a side line) */
  int64_t n_sources;    /* far-field point sources (n_tri * len_q) */
  int32_t max_depth;
  int32_t gpu_launches; /* kernels launched by this call */
  double t_list_ms;     /* device time: near-field list build (K3) */
  double t_far_ms;      /* device time: strengths + far sum (K1, K2): T_F */
  double t_near_ms;     /* device time: near pairs (K4): T_N */
  double t_self_ms;     /* device time: self pairs (K5): T_S */
  double t_total_ms;    /* device time of the whole evaluation */
  double t_sources_ms;  /* device time of K1 alone */
  double t_far_kernel_ms; /* device time of K2 (far sum + its fixed-order reduction) */
  int32_t far_method;   /* 0 direct, 1 FMM */
  int32_t fmm_levels;   /* leaf level of the FMM quadtree */
  int64_t fmm_outside;  /* targets outside the FMM root box (summed directly) */
  double t_pair_ms;     /* device time of the pair stage: near (K4), self (K5) and the
                           point sums, which run side by side on two streams */
} vp_stats;

/* context (device = CUDA ordinal) */
int vp_create(int device, vp_ctx** out);
void vp_destroy(vp_ctx* ctx);
const char* vp_last_error(const vp_ctx* ctx);

/* TriMesh restricted to straight triangles: vertices
 * [n_vert*2], triangles [n_tri*3] counter-clockwise.  Affine element map
 * rho_T(xi,eta) = v0 + xi (v1-v0) + eta (v2-v0). */
int vp_set_mesh(vp_ctx* ctx, int64_t n_vert, const double* vxy, int64_t n_tri,
                const int32_t* tri);

/* Curved (blending-map) elements; replaces the reference's
 * per-element `kind/curve/s_a/s_b` fields of TriMesh (SPEC.md:171-179,
 * :339-376) with a Legendre series per curve.  curve_id[e] >= 0 marks
 * triangle e as curved: its vertices are (gamma(L), gamma(0), O) and its side
 * from vertex 1 to vertex 0 is gamma(tau L) = sum_n (cx, cy)[id*(deg+1) + n]
 * P_n(2 tau - 1), tau in [0, 1], of arc length len[id].  The map is the
 * blending map of PAPER.md eq. for:blend; sources, lists (Newton locate),
 * near and self quadrature follow it.  curve_id == NULL clears; a new mesh
 * clears.  Call after vp_set_mesh. */
int vp_set_curves(vp_ctx* ctx, const int32_t* curve_id, int deg, int64_t n_curves, const double* cx,
                  const double* cy, const double* len);

/* Rules + tolerance; builds the per-element near-field models
 * (build_model) on the host so list predicates are
 * bit-reproducible, and the element bins used by the list build.
 * near_eval accepts a sub-simplex once rho_d = rho0(N_n) 4^{-d/N_n} <= 1, so
 * an element's leaves are at most d* deep; leaf path codes hold 29 levels
 * (the reference allows 40), so an element with d* > 29
 * (rho0 of the N_n model above 4^{29/12} = 28.5: eps far below the element's
 * weight) is refused here with status 2.  Every BASELINE configuration has
 * d* <= 19. */
int vp_set_rules(vp_ctx* ctx, const vp_rules* rules);

/* Density as order-p Koornwinder coefficients per triangle, [n_tri * M_p],
 * graded order (koornwinder.hpp:12-21); p <= 12. */
int vp_set_density(vp_ctx* ctx, int p, const double* coeffs);

/* Near-field lists (locate + nearby + in_near_field, SPEC.md:368-386,
 * :450-458): self_out[t] = S(t) (-1 outside), CSR offsets [n_tgt+1] and
 * ascending element ids.  With ids_out == NULL only *n_ids is returned. */
int vp_build_nearlist(vp_ctx* ctx, int64_t n_tgt, const double* txy, int32_t* self_out,
                      int64_t* offsets_out, int32_t* ids_out, int64_t ids_cap,
                      int64_t* n_ids);

/* Full evaluation (evaluate_field phases 1-2 with the direct far path,
 * SPEC.md:582-590, :618): u[t] = far sum + sum_{N(t)} (near_eval - point
 * sum) + (self_eval - point sum).  Host arrays in and out. */
int vp_evaluate(vp_ctx* ctx, int64_t n_tgt, const double* txy, double* u_out, vp_stats* st);

/* Same with device-resident targets and output (pointers on ctx's device),
 * for callers that keep data in HBM; `stream` may be NULL (ctx stream). */
int vp_evaluate_device(vp_ctx* ctx, int64_t n_tgt, const double* d_txy, double* d_u,
                       void* stream, vp_stats* st);

/* Stream-ordered evaluation from a captured CUDA graph.  The first call for
 * a (targets, output, configuration) triple runs one eager evaluation, which
 * fixes every host-side size (list and leaf totals, overflow counts, FMM
 * outside targets: they depend on the targets, mesh, rules and models, never
 * on the density), then captures the same evaluation with no host round
 * trip into a graph; every call launches that graph on `stream` (NULL: ctx
 * stream) and returns at once.  The graph reads d_txy, the density
 * coefficients and the rules in place: replays stay valid across
 * vp_set_density of the same order, and are re-captured after any other
 * vp_set_* or a different (n_tgt, d_txy, d_u).  The caller must not change
 * the targets' values in place without a new pointer.  Errors of a replay
 * and its counters: vp_graph_status. */
int vp_evaluate_graph(vp_ctx* ctx, int64_t n_tgt, const double* d_txy, double* d_u, void* stream);
/* Waits for `stream` (NULL: ctx stream) and reports the last replay's device
 * error flags (status 2 as vp_evaluate) and counters (no device times). */
int vp_graph_status(vp_ctx* ctx, void* stream, vp_stats* st);

/* Far field only (fmm_eval --direct): u_far[t] =
 * sum_j q_j log r_tj^2, q_j = w_j |J| f_j / (4 pi); coincident pairs give 0. */
int vp_far_field(vp_ctx* ctx, int64_t n_tgt, const double* txy, double* u_far);

/* Point sources of the far field (ChargeSystem):
 * sx, sy, q [n_tri * len_q], element-major. */
int vp_sources(vp_ctx* ctx, double* sx, double* sy, double* q);

/* Per-pair corrections for explicit (target, element) pairs: near_eval
 * and the point sum it replaces; and self_eval
 * for targets inside `elem`.  leaves/panels per pair. */
int vp_near_pairs(vp_ctx* ctx, int64_t n_pairs, const double* txy, const int32_t* elem,
                  double* val, double* sub, int64_t* leaves);
int vp_self_pairs(vp_ctx* ctx, int64_t n_pairs, const double* txy, const int32_t* elem,
                  double* val, double* sub, int64_t* panels);

/* Far-field method: 0 = direct O(T S) sum (fmm_eval --direct, SPEC.md:618;
 * the default), 1 = 2-D Laplace FMM (fmm_eval; SURVEY.md
 * §8(f1)) with expansion order `order` (0 -> 31, 32 coefficients = one per lane) and about `leaf_size`
 * sources per leaf box (0 -> 40).  Both compute u_far to fp64 parity.
 * 2 = none: vp_evaluate returns the corrections only, sum over N(t) and S(t)
 * of (I_T(t) - point sum), for a caller that supplies its own far field
 * (the subtract-and-add split of SPEC.md:612-615). */
int vp_set_far_method(vp_ctx* ctx, int method, int order, int leaf_size);

/* The FMM order from a far-field tolerance (fmm_eval's eps_fmm):
 * vp_fmm_order_for returns the smallest supported order whose far-field error
 * against the direct sum (relative max-norm, calibrated on the BASELINE
 * configurations) is below eps_fmm: 7, 11, .., 31; below 1e-13 the order
 * stays 31 (error floor 8e-15).  vp_set_fmm_tolerance = vp_set_far_method(ctx,
 * 1, vp_fmm_order_for(eps_fmm), leaf_size); eps_fmm outside (0, 1) is a usage
 * error. */
int vp_fmm_order_for(double eps_fmm);
int vp_set_fmm_tolerance(vp_ctx* ctx, double eps_fmm, int leaf_size);

/* Potential interpolation.  interp_coeffs (rules.hpp:
 * 165-170): per-element Koornwinder coefficients [n_elem * M_p] from values
 * at the M_p reference nodes (ref_x, ref_y) of an interpolation rule, e.g.
 * u at the element's targets; *cond receives the infinity-norm condition
 * number of the Vandermonde (make_interp_rule, rules.hpp:139-156). */
int vp_interp_coeffs(vp_ctx* ctx, int p, const double* ref_x, const double* ref_y, int64_t n_elem,
                     const double* values, double* coeffs, double* cond);

/* field_eval: evaluate the PotentialField (interpolation
 * mesh + coefficients) at points; points outside every element give NaN,
 * elem_out = -1 and are counted in *n_outside. */
int vp_field_eval(vp_ctx* ctx, int64_t n_vert, const double* vxy, int64_t n_tri, const int32_t* tri,
                  int p, const double* coeffs, int64_t n_pts, const double* pts, double* out,
                  int32_t* elem_out, int64_t* n_outside);

/* Near-field model: 0 = precise three-Bernstein-ellipse model (SPEC.md:
 * 411-458, default), 1 = the naive ball baseline (circumscribed circle scaled
 * by ball_factor, 1.5 in SPEC.md:585) for both the lists and the near_eval
 * sub-simplex acceptance (depth capped at 20).  Used for the paper's
 * correction-count comparison (Table near_corr). */
int vp_set_near_model(vp_ctx* ctx, int model, double ball_factor);

/* Near-leaf density cache: w_i f at the N_n-rule nodes of every sub-simplex
 * of depth <= max_depth (-1 disables; default 3) is precomputed per element
 * and shared by all targets, within max_bytes of HBM (0 -> min(48 GiB, a
 * quarter of the free device memory); the depth is lowered until it fits).
 * Values match the recurrence to rounding. */
int vp_set_near_cache(vp_ctx* ctx, int max_depth, int64_t max_bytes);

/* ---- multi-GPU ----
 * Targets are sharded over ranks, one context (usually one process) per GPU,
 * mesh and density replicated on every rank; the only collective is the
 * gather of u (north_star).  NCCL is loaded at run time (libnccl.so.2). */

/* Cost-balanced contiguous split of caller-supplied per-target costs (host
 * only, no device): bounds[r] = the smallest i with sum(cost[0..i)) * world
 * >= r * total; bounds[0] = 0, bounds[world] = n. */
int vp_shard_bounds(int64_t n, const int64_t* cost, int world, int64_t* bounds);

/* Shard plan of a target set: order_out[n_tgt] = the Morton (Z-order)
 * permutation of the targets (16 bits per axis over their bounding box,
 * stable), bounds_out[world+1] = a split of the Morton-ordered targets into
 * contiguous shards of equal estimated cost (FP64 flops: the far field per
 * the far method, |N(t)| near pairs and the self pair, from the near-field
 * list build); shard_cost_out[world] (optional) the cost per shard.  Rank r
 * evaluates targets order_out[bounds[r] .. bounds[r+1]). */
int vp_shard_plan(vp_ctx* ctx, int64_t n_tgt, const double* txy, int world, int32_t* order_out,
                  int64_t* bounds_out, int64_t* shard_cost_out);

#define VP_NCCL_ID_BYTES 128
/* NCCL unique id for vp_comm_init (rank 0 creates it; the caller ships the
 * VP_NCCL_ID_BYTES bytes to the other ranks by its own means). */
int vp_nccl_unique_id(unsigned char* id_out);
/* The context's NCCL communicator: rank `rank` of `world`, on ctx's device. */
int vp_comm_init(vp_ctx* ctx, int world, int rank, const unsigned char* id);
/* All-gather of u: rank r's d_u_local holds targets bounds[r] .. bounds[r+1]
 * of the job; every rank receives the whole u in d_u_all[bounds[world]]
 * (one NCCL broadcast per shard, in a group, straight into place).
 * Stream-ordered on `stream` (NULL: ctx stream). */
int vp_gather(vp_ctx* ctx, const int64_t* bounds, const double* d_u_local, double* d_u_all, void* stream);
/* vp_stats over ranks: counters summed, device times and max_depth maxed. */
int vp_allreduce_stats(vp_ctx* ctx, vp_stats* st);

/* SM count and compute capability of the context's device. */
int vp_device_info(vp_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor);

#ifdef __cplusplus
}
#endif
#endif
