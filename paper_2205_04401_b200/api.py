"""Host-side mirror of the reference's evaluation interface for the hot path.

Names follow the reference specification so a user of the reference finds
the same entry points (SPEC.md module -> here):

  basis      koornwinder size, rules        simplex_rule, gauss_legendre, build_ggq
  nearfield  cn_lookup                      cn_lookup
  element-map / nearfield                   Evaluator.build_nearlist (locate+nearby+in_near_field)
  quadrature-engine                         near_eval / self_eval / far_eval (per pair, GPU)
  fmm-pipeline                              fmm_eval(direct=True), evaluate_field

Every compute call goes through the C-ABI of libvp_b200.so (include/vp.h);
errors map to the reference's exception kinds: UsageError
(std::invalid_argument, code 1), NumericalError (std::runtime_error /
std::domain_error, code 2), DeviceError (code 3, no usable B200).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import VpRules, VpStats, VpsConfigInfo, c_double_p, c_int32_p, c_int64_p


class VolpotError(RuntimeError):
    code = 0


class UsageError(VolpotError, ValueError):
    code = 1


class NumericalError(VolpotError):
    code = 2


class DeviceError(VolpotError):
    code = 3


_ERRS = {1: UsageError, 2: NumericalError, 3: DeviceError}


def _check(rc: int, msg: str):
    if rc != 0:
        raise _ERRS.get(rc, VolpotError)(f"[{rc}] {msg}")


def _d(a):
    return a.ctypes.data_as(c_double_p)


def _i32(a):
    return a.ctypes.data_as(c_int32_p)


def _i64(a):
    return a.ctypes.data_as(c_int64_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _setup_err():
    return _lib.lib().vps_last_error().decode()


# ---------------------------------------------------------------------------
# basis / rules (host setup)

def koorn_size(p: int) -> int:
    """(p+1)(p+2)/2 (koornwinder.hpp:20)."""
    return (p + 1) * (p + 2) // 2


def koorn_index(m: int, n: int) -> int:
    """graded index n(n+1)/2 + m (koornwinder.hpp:21)."""
    return n * (n + 1) // 2 + m


def cn_lookup(n: int) -> float:
    """C_N calibration.  Orders below
    12 are clamped to C_12 = 12 (policy SURVEY.md §9.3; the reference errors)."""
    kn = [12, 20, 25, 30, 40, 50]
    kc = [12.0, 6.8, 3.0, 2.5, 2.0, 1.0]
    if n <= 12:
        return 12.0
    if n >= 50:
        return 1.0
    for i in range(5):
        if n == kn[i]:
            return kc[i]
        if kn[i] < n < kn[i + 1]:
            f = float(n - kn[i]) / float(kn[i + 1] - kn[i])
            return kc[i] + (kc[i + 1] - kc[i]) * f
    return 1.0


def simplex_rule(order: int):
    """(x, y, w) of the order-`order` collapsed Gauss-Jacobi rule on Delta^1."""
    L = _lib.lib()
    n = ctypes.c_int()
    _check(L.vps_simplex_rule(order, ctypes.byref(n), None, None, None), _setup_err())
    x, y, w = (np.zeros(n.value) for _ in range(3))
    _check(L.vps_simplex_rule(order, ctypes.byref(n), _d(x), _d(y), _d(w)), _setup_err())
    return x, y, w


def quad_rule(order: int):
    """(x, y, w) of the evaluation's far / near rule of order `order`
    (load_far_rule, rules.hpp:121-125): the repository's own fully symmetric
    rule where one is tabulated (degrees 6, 10, 12), else simplex_rule."""
    L = _lib.lib()
    n = ctypes.c_int()
    _check(L.vps_quad_rule(order, ctypes.byref(n), None, None, None), _setup_err())
    x, y, w = (np.zeros(n.value) for _ in range(3))
    _check(L.vps_quad_rule(order, ctypes.byref(n), _d(x), _d(y), _d(w)), _setup_err())
    return x, y, w


def gauss_legendre(n: int):
    """Gauss-Legendre on [-1, 1] (gauss.hpp:17-46)."""
    x, w = np.zeros(n), np.zeros(n)
    _check(_lib.lib().vps_gauss_legendre(n, _d(x), _d(w)), _setup_err())
    return x, w


def build_ggq(ng: int):
    """Radial GGQ rule with ng+1 nodes (ggq.hpp:96-182); returns (r, w, residual)."""
    r, w, res = np.zeros(ng + 1), np.zeros(ng + 1), ctypes.c_double()
    _check(_lib.lib().vps_ggq(ng, _d(r), _d(w), ctypes.byref(res)), _setup_err())
    return r, w, res.value


def lattice_nodes(p: int):
    m = koorn_size(p)
    x, y = np.zeros(m), np.zeros(m)
    _check(_lib.lib().vps_lattice_nodes(p, _d(x), _d(y)), _setup_err())
    return x, y


@dataclass
class Rules:
    """Everything vp_set_rules needs (far rule of order q, near rule N_n,
    GL N_l, GGQ N_g, tolerance eps).  Defaults mirror SPEC.md:733."""
    q: int
    far: tuple
    n_n: int
    near: tuple
    gl: tuple
    n_g: int
    ggq: tuple
    eps: float

    def as_struct(self) -> VpRules:
        self._keep = [np.ascontiguousarray(a, dtype=np.float64)
                      for a in (*self.far, *self.near, *self.gl, *self.ggq)]
        k = self._keep
        return VpRules(q=self.q, len_q=len(k[0]), far_x=_d(k[0]), far_y=_d(k[1]), far_w=_d(k[2]),
                       n_n=self.n_n, len_n=len(k[3]), near_x=_d(k[3]), near_y=_d(k[4]),
                       near_w=_d(k[5]), n_l=len(k[6]), gl_x=_d(k[6]), gl_w=_d(k[7]),
                       n_g=self.n_g, ggq_r=_d(k[8]), ggq_w=_d(k[9]), eps=self.eps)


def make_rules(q: int, n_n: int = 12, n_l: int = 16, n_g: int = 8, eps: float = 1e-12) -> Rules:
    r, w, _ = build_ggq(n_g)
    return Rules(q=q, far=quad_rule(q), n_n=n_n, near=quad_rule(n_n), gl=gauss_legendre(n_l),
                 n_g=n_g, ggq=(r, w), eps=eps)


def project_density(vxy, tri, p: int, kind: int, params=()):
    """Per-triangle Koornwinder coefficients of an analytic density (L2 projection)."""
    vxy = _f64(vxy, (-1, 2))
    tri = np.ascontiguousarray(tri, dtype=np.int32).reshape(-1, 3)
    prm = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(-1))
    if prm.size == 0:
        prm = np.zeros(1)
    out = np.zeros((tri.shape[0], koorn_size(p)))
    _check(_lib.lib().vps_project_density(vxy.shape[0], _d(vxy), tri.shape[0], _i32(tri), p, kind,
                                          _d(prm), len(params), _d(out)), _setup_err())
    return out


def density_eval(kind: int, params, x: float, y: float) -> float:
    prm = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(-1))
    if prm.size == 0:
        prm = np.zeros(1)
    return _lib.lib().vps_density_eval(kind, _d(prm), len(params), x, y)


F_CONST, F_SQUARE, F_GAUSS, F_BUMPS, F_COSSIN, F_LINEAR = range(6)


@dataclass
class Problem:
    """A mesh, density coefficients, targets and rules (one BASELINE config)."""
    config: int
    vxy: np.ndarray
    tri: np.ndarray
    txy: np.ndarray
    coeffs: np.ndarray
    p: int
    q: int
    eps: float
    seed: int
    density_kind: int
    params: np.ndarray
    staggered: bool
    rules: Rules = field(default=None)

    @property
    def n_tri(self):
        return self.tri.shape[0]

    @property
    def n_tgt(self):
        return self.txy.shape[0]


def config_info(cfg: int, q_override: int = 0, seed: int = 0) -> dict:
    info = VpsConfigInfo()
    _check(_lib.lib().vps_config_info_get(cfg, q_override, seed, ctypes.byref(info)), _setup_err())
    return {"n_vert": info.n_vert, "n_tri": info.n_tri, "n_tgt": info.n_tgt, "p": info.p,
            "q": info.q, "eps": info.eps, "density_kind": info.density_kind,
            "params": np.array(info.params[:info.n_params]), "staggered": bool(info.staggered)}


def load_config(cfg: int, q_override: int = 0, seed: int = 0, with_rules: bool = True) -> Problem:
    """Synthetic BASELINE.json config `cfg` (1..5) from the seeded generators."""
    I = config_info(cfg, q_override, seed)
    vxy = np.zeros((I["n_vert"], 2))
    tri = np.zeros((I["n_tri"], 3), dtype=np.int32)
    txy = np.zeros((I["n_tgt"], 2))
    coeffs = np.zeros((I["n_tri"], koorn_size(I["p"])))
    _check(_lib.lib().vps_config_fill(cfg, q_override, seed, _d(vxy), _i32(tri), _d(txy), _d(coeffs)),
           _setup_err())
    pr = Problem(config=cfg, vxy=vxy, tri=tri, txy=txy, coeffs=coeffs, p=I["p"], q=I["q"], eps=I["eps"],
                 seed=seed, density_kind=I["density_kind"], params=I["params"],
                 staggered=I["staggered"])
    if with_rules:
        pr.rules = make_rules(pr.q, eps=pr.eps)
    return pr


@dataclass
class Curves:
    """Curved (blending-map) elements: curve_id[e] >= 0 marks element e as
    curved, vertex order (gamma(L), gamma(0), O); its side is
    gamma(tau L) = sum_n (cx, cy)[curve_id, n] P_n(2 tau - 1)."""
    curve_id: np.ndarray
    deg: int
    cx: np.ndarray
    cy: np.ndarray
    length: np.ndarray


def circle_arc(cx, cy, R, th0, th1, deg=16):
    gx, gy, ln = np.zeros(deg + 1), np.zeros(deg + 1), ctypes.c_double()
    _check(_lib.lib().vps_circle_arc(cx, cy, R, th0, th1, deg, _d(gx), _d(gy), ctypes.byref(ln)), _setup_err())
    return gx, gy, ln.value


class BoundaryCurve:
    """Closed boundary curve with its arc-length parametrisation (the
    reference's ParamCurve + ArcLengthCurve, curve.hpp:16-332), host C++."""

    CIRCLE, ELLIPSE, WOBBLY, HERMITE, ARC = 0, 1, 2, 3, 4

    def __init__(self, kind, params):
        self._L = _lib.lib()
        prm = np.ascontiguousarray(params, dtype=np.float64).ravel()
        h = ctypes.c_void_p()
        _check(self._L.vps_curve_create(kind, _d(prm), prm.size, ctypes.byref(h)),
               self._L.vps_curve_last_error().decode())
        self._h = h
        self.kind = kind
        self.length = self._L.vps_curve_length(h)
        self.ccw = bool(self._L.vps_curve_ccw(h))

    @classmethod
    def circle(cls, cx=0.0, cy=0.0, r=1.0):
        return cls(cls.CIRCLE, [cx, cy, r])

    @classmethod
    def ellipse(cls, a, b):
        return cls(cls.ELLIPSE, [a, b])

    @classmethod
    def wobbly(cls, a, b, k):
        return cls(cls.WOBBLY, [a, b, k])

    @classmethod
    def hermite(cls, samples):
        """samples: rows `t x y dx dy` (the reference's curve text format)."""
        return cls(cls.HERMITE, np.asarray(samples, dtype=np.float64).reshape(-1, 5))

    @classmethod
    def arc(cls, cx, cy, r, th0, th1):
        return cls(cls.ARC, [cx, cy, r, th0, th1])

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.vps_curve_destroy(self._h)
            self._h = None

    def param(self, s):
        t = ctypes.c_double()
        _check(self._L.vps_curve_param(self._h, float(s), ctypes.byref(t)), self._L.vps_curve_last_error().decode())
        return t.value

    def points(self, s):
        """(Gamma(s), unit tangent, Gamma''(s)) at arc lengths s."""
        s = np.ascontiguousarray(np.atleast_1d(s), dtype=np.float64)
        xy, tg, dd = np.zeros((s.size, 2)), np.zeros((s.size, 2)), np.zeros((s.size, 2))
        _check(self._L.vps_curve_points(self._h, s.size, _d(s), _d(xy), _d(tg), _d(dd)),
               self._L.vps_curve_last_error().decode())
        return xy, tg, dd

    def closest(self, xy):
        xy = _f64(xy, (-1, 2))
        s, dist = np.zeros(xy.shape[0]), np.zeros(xy.shape[0])
        _check(self._L.vps_curve_closest(self._h, xy.shape[0], _d(xy), _d(s), _d(dist)),
               self._L.vps_curve_last_error().decode())
        return s, dist

    def segment(self, s_from, s_to, deg=16):
        gx, gy, ln = np.zeros(deg + 1), np.zeros(deg + 1), ctypes.c_double()
        _check(self._L.vps_curve_segment(self._h, float(s_from), float(s_to), deg, _d(gx), _d(gy), ctypes.byref(ln)),
               self._L.vps_curve_last_error().decode())
        return gx, gy, ln.value


def curves_from_annotation(vxy, tri, meta, curves, deg=16):
    """Curved elements from the reference's TriMesh annotation (SPEC.md:171,
    mesh file `e i j k kind opp curve s_a s_b`): meta rows (kind, opp, curve,
    s_a, s_b), kind 0 straight.  Returns (tri reordered to (gamma(L), gamma(0),
    O) for curved elements, Curves)."""
    vxy = np.asarray(vxy, dtype=np.float64)
    tri = np.array(tri, dtype=np.int32).reshape(-1, 3).copy()
    cid = -np.ones(len(tri), dtype=np.int32)
    cxs, cys, lens = [], [], []
    for e, row in enumerate(meta):
        kind, opp, ci, sa, sb = int(row[0]), int(row[1]), int(row[2]), float(row[3]), float(row[4])
        if kind == 0:
            continue
        C = curves[ci]
        o = tri[e, opp]
        a, b = tri[e, (opp + 1) % 3], tri[e, (opp + 2) % 3]
        if sb <= sa:
            sb += C.length
        pa, pb = C.points([sa, sb])[0]
        # which stored vertex is gamma(s_a)
        if np.hypot(*(vxy[a] - pa)) + np.hypot(*(vxy[b] - pb)) > np.hypot(*(vxy[b] - pa)) + np.hypot(*(vxy[a] - pb)):
            a, b = b, a
        if max(np.hypot(*(vxy[a] - pa)), np.hypot(*(vxy[b] - pb))) > 1e-10 * max(1.0, C.length):
            raise UsageError(f"element {e}: curved side endpoints differ from gamma(s_a), gamma(s_b) by > 1e-10")
        det = (vxy[b, 0] - vxy[a, 0]) * (vxy[o, 1] - vxy[a, 1]) - (vxy[o, 0] - vxy[a, 0]) * (vxy[b, 1] - vxy[a, 1])
        if det > 0:  # (Gamma(s_a), Gamma(s_b), O) counter-clockwise: gamma(sigma) = Gamma(s_b - sigma)
            tri[e] = (a, b, o)
            gx, gy, ln = C.segment(sb, sa, deg)
        else:
            tri[e] = (b, a, o)
            gx, gy, ln = C.segment(sa, sb, deg)
        cid[e] = len(lens)
        cxs.append(gx)
        cys.append(gy)
        lens.append(ln)
    if not lens:
        return tri, None
    return tri, Curves(cid, deg, np.array(cxs), np.array(cys), np.array(lens))


def annotate_boundary(vxy, tri, curves, tol=1e-10):
    """annotate_boundary: every boundary edge (an edge of
    exactly one triangle) becomes the curved side of its triangle, its
    endpoints resolved on the nearest curve by closest point.  Returns
    (meta rows (kind, opp, curve, s_a, s_b), vxy with the boundary vertices
    snapped onto the curves)."""
    vxy = np.array(vxy, dtype=np.float64).reshape(-1, 2)
    tri = np.asarray(tri, dtype=np.int64).reshape(-1, 3)
    edges = {}
    for e, t in enumerate(tri):
        for k in range(3):
            a, b = int(t[(k + 1) % 3]), int(t[(k + 2) % 3])
            edges.setdefault((min(a, b), max(a, b)), []).append((e, k))
    bnd = sorted({v for (a, b), els in edges.items() if len(els) == 1 for v in (a, b)})
    bv = np.array(bnd, dtype=np.int64)
    best_c = np.full(len(bv), -1)
    best_s = np.zeros(len(bv))
    best_d = np.full(len(bv), np.inf)
    for ci, C in enumerate(curves):
        s, d = C.closest(vxy[bv])
        upd = d < best_d
        best_c[upd], best_s[upd], best_d[upd] = ci, s[upd], d[upd]
    scale = max(max(C.length for C in curves), 1.0)
    if (best_d > tol * scale).any():
        raise UsageError("annotate_boundary: boundary vertex farther than tol from every curve")
    vc = dict(zip(bnd, best_c))
    vs = dict(zip(bnd, best_s))
    for ci, C in enumerate(curves):
        sel = best_c == ci
        if sel.any():
            vxy[bv[sel]] = C.points(best_s[sel])[0]
    meta = np.zeros((len(tri), 5))
    for (a, b), els in edges.items():
        if len(els) != 1:
            continue
        e, k = els[0]
        if meta[e, 0] != 0:
            raise UsageError(f"annotate_boundary: element {e} has two boundary edges")
        if vc[a] != vc[b]:
            raise UsageError("annotate_boundary: boundary edge whose endpoints resolve to different curves")
        C = curves[vc[a]]
        sa, sb = vs[a], vs[b]
        d = (sb - sa) % C.length
        if d > C.length / 2:  # the short way round: s_a -> s_b increasing
            sa, sb = sb, sa
        meta[e] = (1, k, vc[a], sa, sb)
    return meta, vxy


def curve_boundary_of_disk(vxy, tri, R=1.0, deg=16, tol=1e-12):
    """Turn every triangle of a disk mesh with an edge on |x| = R into a
    curved element on the exact circle (vertices reordered to
    (gamma(L), gamma(0), O), counter-clockwise).  Returns (tri, Curves)."""
    vxy = np.asarray(vxy, dtype=np.float64)
    tri = np.array(tri, dtype=np.int32).reshape(-1, 3).copy()
    on = np.abs(np.hypot(vxy[:, 0], vxy[:, 1]) - R) <= tol
    cid = -np.ones(len(tri), dtype=np.int32)
    cxs, cys, lens = [], [], []
    for e, t in enumerate(tri):
        flags = on[t]
        if flags.sum() != 2:
            continue
        k = int(np.nonzero(~flags)[0][0])  # the interior vertex O
        a, b, o = t[(k + 1) % 3], t[(k + 2) % 3], t[k]  # CCW (A, B, O)
        tri[e] = (a, b, o)
        tha = np.arctan2(vxy[a, 1], vxy[a, 0])
        thb = np.arctan2(vxy[b, 1], vxy[b, 0])
        if thb < tha:
            thb += 2 * np.pi
        gx, gy, ln = circle_arc(0.0, 0.0, R, thb, tha, deg)  # gamma(0) = B -> gamma(L) = A
        cid[e] = len(lens)
        cxs.append(gx)
        cys.append(gy)
        lens.append(ln)
    return tri, Curves(cid, deg, np.array(cxs), np.array(cys), np.array(lens))


# ---------------------------------------------------------------------------
# evaluator (GPU, through the C-ABI)

class Evaluator:
    """One context on one CUDA device (one process per GPU)."""

    def __init__(self, device: int = 0):
        self._L = _lib.lib()
        h = ctypes.c_void_p()
        rc = self._L.vp_create(device, ctypes.byref(h))
        if rc != 0:
            raise _ERRS.get(rc, VolpotError)(
                f"[{rc}] vp_create(device={device}) failed: no usable sm_100 device "
                "(there is no CPU fallback)")
        self._h = h
        self.device = device
        self.p = None
        self.n_tri = 0

    def _err(self):
        return self._L.vp_last_error(self._h).decode()

    def close(self):
        if getattr(self, "_h", None):
            self._L.vp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_mesh(self, vxy, tri):
        self._vxy = _f64(vxy, (-1, 2))
        self._tri = np.ascontiguousarray(tri, dtype=np.int32).reshape(-1, 3)
        _check(self._L.vp_set_mesh(self._h, self._vxy.shape[0], _d(self._vxy), self._tri.shape[0],
                                   _i32(self._tri)), self._err())
        self.n_tri = self._tri.shape[0]

    def set_curves(self, curves: "Curves | None"):
        """Curved (blending-map) elements; None clears."""
        if curves is None:
            _check(self._L.vp_set_curves(self._h, None, 0, 0, None, None, None), self._err())
            return
        self._cid = np.ascontiguousarray(curves.curve_id, dtype=np.int32)
        self._ccx = np.ascontiguousarray(curves.cx, dtype=np.float64)
        self._ccy = np.ascontiguousarray(curves.cy, dtype=np.float64)
        self._cl = np.ascontiguousarray(curves.length, dtype=np.float64)
        _check(self._L.vp_set_curves(self._h, _i32(self._cid), curves.deg, self._cl.size, _d(self._ccx),
                                     _d(self._ccy), _d(self._cl)), self._err())

    def set_rules(self, rules: Rules):
        self._rules_struct = rules.as_struct()
        self._rules = rules
        _check(self._L.vp_set_rules(self._h, ctypes.byref(self._rules_struct)), self._err())

    def set_far_method(self, method: str = "direct", order: int = 0, leaf_size: int = 0):
        """'direct' (O(T S) sum, default), 'fmm' (2-D Laplace FMM)
        or 'none' (evaluate returns the near/self corrections only, for a caller
        that supplies its own far field: SPEC.md:612-615's subtract-and-add)."""
        m = {"direct": 0, "fmm": 1, "none": 2}[method]
        _check(self._L.vp_set_far_method(self._h, m, order, leaf_size), self._err())

    def set_fmm_tolerance(self, eps_fmm: float, leaf_size: int = 0):
        """FMM far field with the order chosen from eps_fmm (fmm_eval's
        tolerance); see fmm_order_for."""
        _check(self._L.vp_set_fmm_tolerance(self._h, float(eps_fmm), leaf_size), self._err())

    def set_near_model(self, model: str = "precise", ball_factor: float = 1.5):
        """'precise' (Bernstein ellipses, default) or 'ball' (SPEC.md:585 baseline)."""
        m = {"precise": 0, "ball": 1}[model]
        _check(self._L.vp_set_near_model(self._h, m, ball_factor), self._err())

    def set_near_cache(self, max_depth: int = 3, max_bytes: int = 0):
        """Per-element cache of near-rule densities for sub-simplices of depth
        <= max_depth (-1 disables)."""
        _check(self._L.vp_set_near_cache(self._h, max_depth, max_bytes), self._err())

    def set_density(self, p: int, coeffs):
        c = _f64(coeffs)
        _check(self._L.vp_set_density(self._h, p, _d(c)), self._err())
        self.p = p

    def load(self, pr: Problem):
        self.set_mesh(pr.vxy, pr.tri)
        self.set_rules(pr.rules)
        self.set_density(pr.p, pr.coeffs)
        return self

    def build_nearlist(self, txy):
        """(S, offsets, ids): S(t) (-1 outside), CSR of N(t) ascending."""
        t = _f64(txy, (-1, 2))
        n = t.shape[0]
        nids = ctypes.c_int64()
        self_ = np.zeros(n, dtype=np.int32)
        off = np.zeros(n + 1, dtype=np.int64)
        _check(self._L.vp_build_nearlist(self._h, n, _d(t), _i32(self_), _i64(off), None, 0,
                                         ctypes.byref(nids)), self._err())
        ids = np.zeros(max(nids.value, 1), dtype=np.int32)
        _check(self._L.vp_build_nearlist(self._h, n, _d(t), _i32(self_), _i64(off), _i32(ids),
                                         ids.size, ctypes.byref(nids)), self._err())
        return self_, off, ids[:nids.value]

    def evaluate(self, txy):
        """u at the targets and the run statistics (evaluate_field core)."""
        t = _f64(txy, (-1, 2))
        u = np.zeros(t.shape[0])
        st = VpStats()
        _check(self._L.vp_evaluate(self._h, t.shape[0], _d(t), _d(u), ctypes.byref(st)), self._err())
        return u, st.as_dict()

    def evaluate_device(self, n: int, d_txy: int, d_u: int, stream: int = 0):
        st = VpStats()
        _check(self._L.vp_evaluate_device(self._h, n, ctypes.c_void_p(d_txy), ctypes.c_void_p(d_u),
                                          ctypes.c_void_p(stream or None), ctypes.byref(st)),
               self._err())
        return st.as_dict()

    def evaluate_graph(self, n: int, d_txy: int, d_u: int, stream: int = 0):
        """Launch the captured-graph evaluation (vp_evaluate_graph): async, no
        host round trip after the first call for these buffers."""
        _check(self._L.vp_evaluate_graph(self._h, n, ctypes.c_void_p(d_txy), ctypes.c_void_p(d_u),
                                         ctypes.c_void_p(stream or None)), self._err())

    def graph_status(self, stream: int = 0) -> dict:
        st = VpStats()
        _check(self._L.vp_graph_status(self._h, ctypes.c_void_p(stream or None), ctypes.byref(st)), self._err())
        return st.as_dict()

    def far_field(self, txy):
        t = _f64(txy, (-1, 2))
        u = np.zeros(t.shape[0])
        _check(self._L.vp_far_field(self._h, t.shape[0], _d(t), _d(u)), self._err())
        return u

    def sources(self):
        n = self.n_tri * len(self._rules.far[0])
        sx, sy, q = np.zeros(n), np.zeros(n), np.zeros(n)
        _check(self._L.vp_sources(self._h, _d(sx), _d(sy), _d(q)), self._err())
        return sx, sy, q

    def _pairs(self, fn, txy, elem):
        t = _f64(txy, (-1, 2))
        e = np.ascontiguousarray(elem, dtype=np.int32).reshape(-1)
        n = t.shape[0]
        val, sub, cnt = np.zeros(n), np.zeros(n), np.zeros(n, dtype=np.int64)
        _check(fn(self._h, n, _d(t), _i32(e), _d(val), _d(sub), _i64(cnt)), self._err())
        return val, sub, cnt

    def interp_coeffs(self, p: int, ref_x, ref_y, values):
        """Per-element Koornwinder coefficients from values at the M_p reference
        nodes (interp_coeffs, rules.hpp:165-170); returns (coeffs, condition)."""
        rx, ry = _f64(ref_x), _f64(ref_y)
        v = _f64(values).reshape(-1, koorn_size(p))
        out = np.zeros_like(v)
        cond = ctypes.c_double()
        _check(self._L.vp_interp_coeffs(self._h, p, _d(rx), _d(ry), v.shape[0], _d(v), _d(out),
                                        ctypes.byref(cond)), self._err())
        return out, cond.value

    def field_eval(self, vxy, tri, p: int, coeffs, pts, allow_outside: bool = False):
        """Evaluate a PotentialField at points (field_eval)."""
        v = _f64(vxy, (-1, 2))
        t = np.ascontiguousarray(tri, dtype=np.int32).reshape(-1, 3)
        c = _f64(coeffs)
        x = _f64(pts, (-1, 2))
        out = np.zeros(x.shape[0])
        eo = np.zeros(x.shape[0], dtype=np.int32)
        nout = ctypes.c_int64()
        _check(self._L.vp_field_eval(self._h, v.shape[0], _d(v), t.shape[0], _i32(t), p, _d(c), x.shape[0],
                                     _d(x), _d(out), _i32(eo), ctypes.byref(nout)), self._err())
        if nout.value and not allow_outside:
            raise NumericalError(f"[2] field_eval: {nout.value} point(s) outside domain")
        return out, eo

    # ---- multi-GPU: shard plan + the library's NCCL gather
    def shard_plan(self, txy, world: int):
        """(order, bounds, shard_cost): Morton permutation of the targets and a
        cost-balanced split into `world` contiguous shards (vp_shard_plan)."""
        t = _f64(txy, (-1, 2))
        order = np.zeros(t.shape[0], dtype=np.int32)
        bounds = np.zeros(world + 1, dtype=np.int64)
        cost = np.zeros(world, dtype=np.int64)
        _check(self._L.vp_shard_plan(self._h, t.shape[0], _d(t), world, _i32(order), _i64(bounds), _i64(cost)),
               self._err())
        return order, bounds, cost

    def comm_init(self, world: int, rank: int, uid: bytes):
        """Join the library's NCCL communicator (uid from nccl_unique_id() on rank 0)."""
        if len(uid) != NCCL_ID_BYTES:
            raise UsageError(f"[1] comm_init: the unique id has {NCCL_ID_BYTES} bytes")
        _check(self._L.vp_comm_init(self._h, world, rank, uid), self._err())

    def gather(self, bounds, d_u_local: int, d_u_all: int, stream: int = 0):
        """All-gather of u over the communicator (device pointers, stream-ordered)."""
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        _check(self._L.vp_gather(self._h, _i64(b), ctypes.c_void_p(d_u_local), ctypes.c_void_p(d_u_all),
                                 ctypes.c_void_p(stream or None)), self._err())

    def allreduce_stats(self, st: dict) -> dict:
        s = VpStats(**{k: st[k] for k, _ in VpStats._fields_})
        _check(self._L.vp_allreduce_stats(self._h, ctypes.byref(s)), self._err())
        return s.as_dict()

    def near_pairs(self, txy, elem):
        """near_eval(T, t), the point sum it replaces, and leaf counts."""
        return self._pairs(self._L.vp_near_pairs, txy, elem)

    def self_pairs(self, txy, elem):
        """self_eval(T, t), the point sum it replaces, and panel counts."""
        return self._pairs(self._L.vp_self_pairs, txy, elem)


NCCL_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0), to be shipped to the other ranks."""
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    rc = _lib.lib().vp_nccl_unique_id(buf)
    if rc != 0:
        raise DeviceError(f"[{rc}] vp_nccl_unique_id: NCCL unavailable")
    return buf.raw


def shard_bounds(cost, world: int) -> np.ndarray:
    """Cost-balanced contiguous split of per-target costs (vp_shard_bounds, host only)."""
    c = np.ascontiguousarray(cost, dtype=np.int64)
    b = np.zeros(world + 1, dtype=np.int64)
    rc = _lib.lib().vp_shard_bounds(c.size, _i64(c), world, _i64(b))
    if rc != 0:
        raise UsageError("[1] shard_bounds: need world >= 1 and non-negative costs")
    return b


def evaluate_field(pr: Problem, targets=None, device: int = 0):
    """evaluate_field, direct far path: potentials at the
    targets plus statistics c, s_n, s_l and the device-time split."""
    with Evaluator(device) as ev:
        ev.load(pr)
        u, st = ev.evaluate(pr.txy if targets is None else targets)
    n = max(st["n_targets"], 1)
    st["c"] = (st["n_near_pairs"] + st["n_self"]) / n
    st["s_n"] = st["n_leaves"] / n
    st["s_l"] = st["n_panels"] / max(st["n_self"], 1)
    return u, st


def fmm_order_for(eps_fmm: float) -> int:
    """The expansion order the library uses for a far-field tolerance eps_fmm."""
    return int(_lib.lib().vp_fmm_order_for(float(eps_fmm)))


def fmm_eval(pr: Problem, targets=None, direct: bool = False, order: int = 0, device: int = 0,
             eps_fmm: float = 0.0):
    """fmm_eval: far field of all quadrature-node charges at
    the targets, by the GPU FMM (order from eps_fmm when given)
    or, with direct=True, the O(N^2) path."""
    with Evaluator(device) as ev:
        ev.load(pr)
        if not direct:
            if eps_fmm > 0.0:
                ev.set_fmm_tolerance(eps_fmm)
            else:
                ev.set_far_method("fmm", order)
        return ev.far_field(pr.txy if targets is None else targets)
