"""ctypes binding of the CPU oracle (liboracle.so) and the reference shim
(oracle/_ref/libvpref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, as the checker.  The
product package (paper_2205_04401_b200) never imports this module.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libvpref.so")

_d_p = ctypes.POINTER(ctypes.c_double)
_i32_p = ctypes.POINTER(ctypes.c_int32)
_i64_p = ctypes.POINTER(ctypes.c_int64)


def _d(a):
    return a.ctypes.data_as(_d_p)


class VpoProblem(ctypes.Structure):
    _fields_ = [
        ("n_vert", ctypes.c_int64), ("vxy", _d_p), ("n_tri", ctypes.c_int64), ("tri", _i32_p),
        ("p", ctypes.c_int), ("coeffs", _d_p),
        ("q", ctypes.c_int), ("len_q", ctypes.c_int), ("far_x", _d_p), ("far_y", _d_p), ("far_w", _d_p),
        ("n_n", ctypes.c_int), ("len_n", ctypes.c_int), ("near_x", _d_p), ("near_y", _d_p),
        ("near_w", _d_p),
        ("n_l", ctypes.c_int), ("gl_x", _d_p), ("gl_w", _d_p),
        ("n_g", ctypes.c_int), ("ggq_r", _d_p), ("ggq_w", _d_p),
        ("eps", ctypes.c_double),
        ("near_model", ctypes.c_int), ("pad_", ctypes.c_int), ("ball_factor", ctypes.c_double),
        ("curve_id", _i32_p), ("curve_deg", ctypes.c_int), ("pad2_", ctypes.c_int),
        ("curve_cx", _d_p), ("curve_cy", _d_p), ("curve_len", _d_p),
    ]


class VpoStats(ctypes.Structure):
    _fields_ = [
        ("n_targets", ctypes.c_int64), ("n_outside", ctypes.c_int64), ("n_near_pairs", ctypes.c_int64),
        ("n_self", ctypes.c_int64), ("n_leaves", ctypes.c_int64), ("n_panels", ctypes.c_int64),
        ("n_rho_le1", ctypes.c_int64), ("n_degenerate", ctypes.c_int64),
        ("max_depth", ctypes.c_int32), ("pad", ctypes.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class VpoConfigInfo(ctypes.Structure):
    _fields_ = [
        ("n_vert", ctypes.c_int64), ("n_tri", ctypes.c_int64), ("n_tgt", ctypes.c_int64),
        ("p", ctypes.c_int), ("q", ctypes.c_int), ("density_kind", ctypes.c_int), ("n_params", ctypes.c_int),
        ("params", ctypes.c_double * 64), ("eps", ctypes.c_double), ("seed", ctypes.c_uint64),
        ("staggered", ctypes.c_int), ("pad", ctypes.c_int),
    ]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(ORACLE_PATH)
        P = ctypes.POINTER(VpoProblem)
        i64, i32, dbl, vp_ = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        sigs = {
            "vpo_last_error": (ctypes.c_char_p, []),
            "vpo_cn_lookup": (dbl, [i32]),
            "vpo_w_edge": (dbl, [i32, _d_p, _d_p, _d_p]),
            "vpo_koornwinder": (i32, [i32, dbl, dbl, _d_p]),
            "vpo_validate_rule": (i32, [i32, i32, _d_p, _d_p, _d_p]),
            "vpo_gauss_legendre": (i32, [i32, _d_p, _d_p]),
            "vpo_quadtree_query": (i32, [i64, _d_p, i32, dbl, dbl, dbl, dbl, _i32_p, i64, _i64_p, _i64_p]),
            "vpo_element_models": (i32, [P, _d_p, _d_p, _d_p]),
            "vpo_nearlist": (i32, [P, i64, _d_p, _i32_p, _i64_p, _i32_p, i64, _i64_p]),
            "vpo_sources": (i32, [P, _d_p, _d_p, _d_p]),
            "vpo_far_sum": (i32, [P, i64, _d_p, i32, _d_p]),
            "vpo_near_pair": (i32, [P, dbl, dbl, ctypes.c_int32, _d_p, _d_p, _i64_p, ctypes.POINTER(ctypes.c_int32)]),
            "vpo_self": (i32, [P, dbl, dbl, ctypes.c_int32, _d_p, _d_p, _i64_p]),
            "vpo_evaluate": (i32, [P, i64, _d_p, i32, _d_p, _d_p, ctypes.POINTER(VpoStats)]),
            "vpo_open": (i32, [P, ctypes.POINTER(ctypes.c_void_p)]),
            "vpo_ctx_evaluate": (i32, [vp_, i64, _d_p, i32, _d_p, _d_p, ctypes.POINTER(VpoStats)]),
            "vpo_close": (None, [vp_]),
            "vpo_inputs_last_error": (ctypes.c_char_p, []),
            "vpo_lattice_nodes": (i32, [i32, _d_p, _d_p]),
            "vpo_gauss_jacobi10": (i32, [i32, _d_p, _d_p]),
            "vpo_simplex_rule": (i32, [i32, ctypes.POINTER(i32), _d_p, _d_p, _d_p]),
            "vpo_quad_rule": (i32, [i32, ctypes.POINTER(i32), _d_p, _d_p, _d_p]),
            "vpo_ggq": (i32, [i32, _d_p, _d_p, ctypes.POINTER(dbl)]),
            "vpo_density_eval": (dbl, [i32, _d_p, i32, dbl, dbl]),
            "vpo_project_density": (i32, [i64, _d_p, i64, _i32_p, i32, i32, _d_p, i32, _d_p]),
            "vpo_config_info_get": (i32, [i32, i32, ctypes.c_uint64, ctypes.POINTER(VpoConfigInfo)]),
            "vpo_config_fill": (i32, [i32, i32, ctypes.c_uint64, _d_p, _i32_p, _d_p, _d_p]),
            "vpo_adaptive_log_integral": (i32, [_d_p, i32, i32, _d_p, i64, _d_p, dbl, i32, _d_p]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ref():
    """The reference's own headers behind an extern "C" shim (None if not built)."""
    global _ref
    if _ref is None and os.path.exists(REF_PATH):
        R = ctypes.CDLL(REF_PATH)
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        R.vpref_koornwinder.argtypes = [i32, dbl, dbl, _d_p]
        R.vpref_gauss_legendre.argtypes = [i32, _d_p, _d_p]
        R.vpref_quadtree_query.argtypes = [i64, _d_p, i32, dbl, dbl, dbl, dbl, _i32_p, i64, _i64_p, _i64_p]
        R.vpref_arclength.argtypes = [i32, _d_p, i32, i64, _d_p, _d_p, _d_p, _d_p, _d_p, ctypes.POINTER(i32)]
        for f in (R.vpref_koornwinder, R.vpref_gauss_legendre, R.vpref_quadtree_query, R.vpref_arclength):
            f.restype = i32
        _ref = R
    return _ref


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().vpo_last_error().decode())


class Oracle:
    """Holds the arrays of one problem and exposes the oracle entry points."""

    def __init__(self, vxy, tri, p, coeffs, rules, near_model=0, ball_factor=1.5, curves=None):
        self.vxy = np.ascontiguousarray(vxy, dtype=np.float64).reshape(-1, 2)
        self.tri = np.ascontiguousarray(tri, dtype=np.int32).reshape(-1, 3)
        self.coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        self.p = p
        self.rules = rules
        self._keep = [np.ascontiguousarray(a, dtype=np.float64)
                      for a in (*rules.far, *rules.near, *rules.gl, *rules.ggq)]
        k = self._keep
        self.pr = VpoProblem(
            n_vert=self.vxy.shape[0], vxy=_d(self.vxy), n_tri=self.tri.shape[0],
            tri=self.tri.ctypes.data_as(_i32_p), p=p, coeffs=_d(self.coeffs),
            q=rules.q, len_q=len(k[0]), far_x=_d(k[0]), far_y=_d(k[1]), far_w=_d(k[2]),
            n_n=rules.n_n, len_n=len(k[3]), near_x=_d(k[3]), near_y=_d(k[4]), near_w=_d(k[5]),
            n_l=len(k[6]), gl_x=_d(k[6]), gl_w=_d(k[7]),
            n_g=rules.n_g, ggq_r=_d(k[8]), ggq_w=_d(k[9]), eps=rules.eps,
            near_model=near_model, ball_factor=ball_factor)
        if curves is not None:
            self._cid = np.ascontiguousarray(curves.curve_id, dtype=np.int32)
            self._ccx = np.ascontiguousarray(curves.cx, dtype=np.float64)
            self._ccy = np.ascontiguousarray(curves.cy, dtype=np.float64)
            self._cl = np.ascontiguousarray(curves.length, dtype=np.float64)
            self.pr.curve_id = self._cid.ctypes.data_as(_i32_p)
            self.pr.curve_deg = curves.deg
            self.pr.curve_cx = _d(self._ccx)
            self.pr.curve_cy = _d(self._ccy)
            self.pr.curve_len = _d(self._cl)

    @classmethod
    def from_problem(cls, pr, near_model=0, ball_factor=1.5):
        return cls(pr.vxy, pr.tri, pr.p, pr.coeffs, pr.rules, near_model, ball_factor)

    def open(self):
        """Persistent context (setup once, evaluate many target batches)."""
        return OracleCtx(self)

    def nearlist(self, txy):
        t = np.ascontiguousarray(txy, dtype=np.float64).reshape(-1, 2)
        n = t.shape[0]
        nids = ctypes.c_int64()
        L = lib()
        _check(L.vpo_nearlist(ctypes.byref(self.pr), n, _d(t), None, None, None, 0, ctypes.byref(nids)))
        s = np.zeros(n, dtype=np.int32)
        off = np.zeros(n + 1, dtype=np.int64)
        ids = np.zeros(max(nids.value, 1), dtype=np.int32)
        _check(L.vpo_nearlist(ctypes.byref(self.pr), n, _d(t), s.ctypes.data_as(_i32_p),
                              off.ctypes.data_as(_i64_p), ids.ctypes.data_as(_i32_p), ids.size,
                              ctypes.byref(nids)))
        return s, off, ids[:nids.value]

    def sources(self):
        n = self.tri.shape[0] * len(self.rules.far[0])
        sx, sy, q = np.zeros(n), np.zeros(n), np.zeros(n)
        _check(lib().vpo_sources(ctypes.byref(self.pr), _d(sx), _d(sy), _d(q)))
        return sx, sy, q

    def far_sum(self, txy, nthreads=0):
        t = np.ascontiguousarray(txy, dtype=np.float64).reshape(-1, 2)
        u = np.zeros(t.shape[0])
        _check(lib().vpo_far_sum(ctypes.byref(self.pr), t.shape[0], _d(t), nthreads, _d(u)))
        return u

    def near_pair(self, tx, ty, elem):
        v, s, lv, dp = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64(), ctypes.c_int32()
        _check(lib().vpo_near_pair(ctypes.byref(self.pr), ctypes.c_double(tx), ctypes.c_double(ty),
                                   int(elem), ctypes.byref(v), ctypes.byref(s), ctypes.byref(lv),
                                   ctypes.byref(dp)))
        return v.value, s.value, lv.value, dp.value

    def self_pair(self, tx, ty, elem):
        v, s, pn = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(lib().vpo_self(ctypes.byref(self.pr), ctypes.c_double(tx), ctypes.c_double(ty), int(elem),
                              ctypes.byref(v), ctypes.byref(s), ctypes.byref(pn)))
        return v.value, s.value, pn.value

    def evaluate(self, txy, nthreads=0):
        t = np.ascontiguousarray(txy, dtype=np.float64).reshape(-1, 2)
        u, uf = np.zeros(t.shape[0]), np.zeros(t.shape[0])
        st = VpoStats()
        _check(lib().vpo_evaluate(ctypes.byref(self.pr), t.shape[0], _d(t), nthreads, _d(u), _d(uf),
                                  ctypes.byref(st)))
        return u, uf, st.as_dict()

    def element_models(self):
        E = self.tri.shape[0]
        rho0, rho0n, ta = np.zeros(E), np.zeros(E), np.zeros(3 * E)
        _check(lib().vpo_element_models(ctypes.byref(self.pr), _d(rho0), _d(rho0n), _d(ta)))
        return rho0, rho0n, ta.reshape(E, 3)


def koornwinder(order, x, y):
    out = np.zeros((order + 1) * (order + 2) // 2)
    _check(lib().vpo_koornwinder(order, ctypes.c_double(x), ctypes.c_double(y), _d(out)))
    return out


def cn_lookup(n):
    return lib().vpo_cn_lookup(n)


def w_edge(x, y, w):
    x, y, w = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, y, w))
    return lib().vpo_w_edge(len(x), _d(x), _d(y), _d(w))


def validate_rule(order, x, y, w):
    x, y, w = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, y, w))
    _check(lib().vpo_validate_rule(order, len(x), _d(x), _d(y), _d(w)))


def gauss_legendre(n):
    x, w = np.zeros(n), np.zeros(n)
    _check(lib().vpo_gauss_legendre(n, _d(x), _d(w)))
    return x, w


def quadtree_query(pts, leaf_cap, rect, use_ref=False):
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    n = ctypes.c_int64()
    vis = ctypes.c_int64()
    L = ref() if use_ref else lib()
    fn = L.vpref_quadtree_query if use_ref else L.vpo_quadtree_query
    args = [pts.shape[0], _d(pts), leaf_cap] + [float(v) for v in rect]
    rc = fn(*args, None, 0, ctypes.byref(n), ctypes.byref(vis))
    if rc:
        raise OracleError(rc, "quadtree query failed")
    out = np.zeros(max(n.value, 1), dtype=np.int32)
    rc = fn(*args, out.ctypes.data_as(_i32_p), out.size, ctypes.byref(n), ctypes.byref(vis))
    if rc:
        raise OracleError(rc, "quadtree query failed")
    return out[:n.value], vis.value


def ref_koornwinder(order, x, y):
    out = np.zeros((order + 1) * (order + 2) // 2)
    rc = ref().vpref_koornwinder(order, ctypes.c_double(x), ctypes.c_double(y), _d(out))
    if rc:
        raise OracleError(rc, "reference koornwinder_eval: point outside the reference simplex")
    return out


def ref_gauss_legendre(n):
    x, w = np.zeros(n), np.zeros(n)
    rc = ref().vpref_gauss_legendre(n, _d(x), _d(w))
    if rc:
        raise OracleError(rc, "reference gauss_legendre failed")
    return x, w


def ref_arclength(kind, params, s):
    """The reference's ArcLengthCurve (curve.hpp:184-332) at arc lengths s:
    (xy, tangent, d2/ds2, length, ccw)."""
    R = ref()
    if R is None:
        raise OracleError(1, "oracle/_ref not built")
    prm = np.ascontiguousarray(params, dtype=np.float64).ravel()
    s = np.ascontiguousarray(np.atleast_1d(s), dtype=np.float64)
    xy, tg, dd = np.zeros((s.size, 2)), np.zeros((s.size, 2)), np.zeros((s.size, 2))
    ln, ccw = ctypes.c_double(), ctypes.c_int()
    rc = R.vpref_arclength(kind, _d(prm), prm.size, s.size, _d(s), _d(xy), _d(tg), _d(dd), ctypes.byref(ln),
                           ctypes.byref(ccw))
    if rc != 0:
        raise OracleError(rc, "reference reparametrize failed")
    return xy, tg, dd, ln.value, bool(ccw.value)


class OracleCtx:
    """vpo_open / vpo_ctx_evaluate / vpo_close: the oracle's setup (element
    models, quadtree, sources) done once for many evaluations."""

    def __init__(self, oracle):
        self.o = oracle  # keeps the problem arrays alive
        h = ctypes.c_void_p()
        _check(lib().vpo_open(ctypes.byref(oracle.pr), ctypes.byref(h)))
        self.h = h

    def evaluate(self, txy, nthreads=0):
        t = np.ascontiguousarray(txy, dtype=np.float64).reshape(-1, 2)
        u, uf = np.zeros(t.shape[0]), np.zeros(t.shape[0])
        st = VpoStats()
        _check(lib().vpo_ctx_evaluate(self.h, t.shape[0], _d(t), nthreads, _d(u), _d(uf), ctypes.byref(st)))
        return u, uf, st.as_dict()

    def close(self):
        if self.h:
            lib().vpo_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# the oracle's own inputs (vp_oracle_inputs.cpp): rules, configurations and
# density coefficients generated without the product library

def _check_in(rc):
    if rc != 0:
        raise OracleError(rc, lib().vpo_inputs_last_error().decode())


def simplex_rule(order):
    n = ctypes.c_int()
    _check_in(lib().vpo_simplex_rule(order, ctypes.byref(n), None, None, None))
    x, y, w = (np.zeros(n.value) for _ in range(3))
    _check_in(lib().vpo_simplex_rule(order, ctypes.byref(n), _d(x), _d(y), _d(w)))
    return x, y, w


def quad_rule(order):
    """The evaluation's far / near rule (symmetric where tabulated, else simplex_rule)."""
    n = ctypes.c_int()
    _check_in(lib().vpo_quad_rule(order, ctypes.byref(n), None, None, None))
    x, y, w = (np.zeros(n.value) for _ in range(3))
    _check_in(lib().vpo_quad_rule(order, ctypes.byref(n), _d(x), _d(y), _d(w)))
    return x, y, w


def gauss_jacobi10(n):
    x, w = np.zeros(n), np.zeros(n)
    _check_in(lib().vpo_gauss_jacobi10(n, _d(x), _d(w)))
    return x, w


def ggq(ng):
    r, w, res = np.zeros(ng + 1), np.zeros(ng + 1), ctypes.c_double()
    _check_in(lib().vpo_ggq(ng, _d(r), _d(w), ctypes.byref(res)))
    return r, w, res.value


def lattice_nodes(p):
    m = (p + 1) * (p + 2) // 2
    x, y = np.zeros(m), np.zeros(m)
    _check_in(lib().vpo_lattice_nodes(p, _d(x), _d(y)))
    return x, y


def project_density(vxy, tri, p, kind, params=()):
    vxy = np.ascontiguousarray(vxy, dtype=np.float64).reshape(-1, 2)
    tri = np.ascontiguousarray(tri, dtype=np.int32).reshape(-1, 3)
    prm = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(-1))
    out = np.zeros((tri.shape[0], (p + 1) * (p + 2) // 2))
    _check_in(lib().vpo_project_density(vxy.shape[0], _d(vxy), tri.shape[0], tri.ctypes.data_as(_i32_p), p, kind,
                                        _d(prm) if prm.size else None, prm.size, _d(out)))
    return out


class OracleRules:
    """Rules in the shape Oracle expects (far, near, gl, ggq tuples), built by
    the oracle's own generators; defaults mirror SPEC.md:733."""

    def __init__(self, q, n_n=12, n_l=16, n_g=8, eps=1e-12):
        self.q, self.n_n, self.n_g, self.eps = q, n_n, n_g, eps
        self.far = quad_rule(q)
        self.near = quad_rule(n_n)
        self.gl = gauss_legendre(n_l)
        r, w, _ = ggq(n_g)
        self.ggq = (r, w)


class OracleProblem:
    """One BASELINE config from the oracle's own seeded generators."""

    def __init__(self, config, q_override=0, seed=0):
        info = VpoConfigInfo()
        _check_in(lib().vpo_config_info_get(config, q_override, seed, ctypes.byref(info)))
        self.config, self.seed = config, seed
        self.p, self.q, self.eps = info.p, info.q, info.eps
        self.density_kind = info.density_kind
        self.params = np.array(info.params[:info.n_params])
        self.staggered = bool(info.staggered)
        self.vxy = np.zeros((info.n_vert, 2))
        self.tri = np.zeros((info.n_tri, 3), dtype=np.int32)
        self.txy = np.zeros((info.n_tgt, 2))
        self.coeffs = np.zeros((info.n_tri, (self.p + 1) * (self.p + 2) // 2))
        _check_in(lib().vpo_config_fill(config, q_override, seed, _d(self.vxy), self.tri.ctypes.data_as(_i32_p),
                                        _d(self.txy), _d(self.coeffs)))
        self.rules = OracleRules(self.q, eps=self.eps)

    @property
    def n_tri(self):
        return self.tri.shape[0]

    @property
    def n_tgt(self):
        return self.txy.shape[0]


def adaptive_log_integral(tri, fkind, pts, coeffs=None, p=0, tol=1e-17, nthreads=0):
    """int_T log|x-y| f(y) dA at exterior points (adaptive subdivision, long
    double; the soundness sweep's oracle)."""
    tri = np.ascontiguousarray(tri, dtype=np.float64).reshape(6)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    c = None if coeffs is None else np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.zeros(pts.shape[0])
    rc = lib().vpo_adaptive_log_integral(_d(tri), fkind, p, _d(c) if c is not None else None, pts.shape[0],
                                         _d(pts), tol, nthreads, _d(out))
    if rc:
        raise OracleError(rc, "adaptive_log_integral: bad arguments")
    return out
