"""GPU parity for curved (blending-map) elements, SURVEY.md §8(f3).

The unit-disk mesh of config 2 with its 256 boundary triangles turned into
curved elements on the exact circle (vp.curve_boundary_of_disk).  Same bar as
tests/test_gpu_parity.py: lists (including the Newton locate of targets that
lie between a chord and its arc) bit-exact, leaf and panel counts identical,
u within 1e-11 relative of the oracle."""
import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from helpers import const_coeffs
from oracle.binding import Oracle

pytestmark = pytest.mark.gpu

REL_TOL = 1e-11


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def ring_targets(n, seed=5):
    """Targets in the boundary layer: between chords and arcs, on the
    circle, and just outside it."""
    rng = np.random.default_rng(seed)
    r = np.concatenate([1.0 - rng.uniform(0, 4e-4, n // 2), 1.0 - rng.uniform(0, 0.05, n // 2 - 8),
                        np.full(4, 1.0), 1.0 + rng.uniform(1e-6, 1e-3, 4)])
    th = rng.uniform(0, 2 * np.pi, r.size)
    return np.stack([r * np.cos(th), r * np.sin(th)], 1)


def make(pr, coeffs, tri, cv, near_model="precise"):
    ev = vp.Evaluator(0)
    ev.set_mesh(pr.vxy, tri)
    ev.set_curves(cv)
    if near_model != "precise":
        ev.set_near_model(near_model)
    ev.set_rules(pr.rules)
    ev.set_density(pr.p, coeffs)
    return ev


@pytest.fixture(scope="module")
def disk():
    pr = vp.load_config(2)
    tri, cv = vp.curve_boundary_of_disk(pr.vxy, pr.tri)
    coeffs = vp.project_density(pr.vxy, tri, pr.p, vp.F_GAUSS, [0.2, -0.1, 3.0])
    txy = np.concatenate([pr.txy[::5], ring_targets(4000)])
    ev = make(pr, coeffs, tri, cv)
    O = Oracle(pr.vxy, tri, pr.p, coeffs, pr.rules, curves=cv)
    yield pr, tri, cv, coeffs, txy, ev, O
    ev.close()


def test_curved_lists_bit_exact(disk):
    pr, tri, cv, coeffs, txy, ev, O = disk
    s_g, off_g, ids_g = ev.build_nearlist(txy)
    s_o, off_o, ids_o = O.nearlist(txy)
    assert np.array_equal(s_g, s_o)
    assert np.array_equal(off_g, off_o)
    assert np.array_equal(ids_g, ids_o)
    # the boundary layer really exercises the curved locate
    ring = txy[-4000:]
    rr = np.hypot(ring[:, 0], ring[:, 1])
    s_ring = s_o[-4000:]
    assert (s_ring[rr < 1.0] >= 0).all()
    assert (s_ring[rr > 1.0 + 1e-9] < 0).all()
    assert (cv.curve_id[s_ring[s_ring >= 0]] >= 0).sum() > 1000


def test_curved_sources_match(disk):
    pr, tri, cv, coeffs, txy, ev, O = disk
    sx, sy, q = ev.sources()
    osx, osy, oq = O.sources()
    assert np.abs(sx - osx).max() <= 1e-15 and np.abs(sy - osy).max() <= 1e-15
    assert rel(q, oq) <= 1e-14


def test_curved_u_and_counts_match_oracle(disk):
    pr, tri, cv, coeffs, txy, ev, O = disk
    sub = np.concatenate([txy[:-4000][::41], txy[-4000:][::7]])
    u_g, st = ev.evaluate(sub)
    u_o, _, sto = O.evaluate(sub)
    assert rel(u_g, u_o) <= REL_TOL
    for k in ("n_near_pairs", "n_leaves", "n_panels", "n_self", "n_outside", "n_rho_le1", "n_degenerate",
              "max_depth"):
        assert st[k] == sto[k], k


def test_curved_pairs_match_oracle(disk):
    pr, tri, cv, coeffs, txy, ev, O = disk
    ring = txy[-4000:][::9]
    s, off, ids = O.nearlist(ring)
    ts = np.repeat(np.arange(len(s)), np.diff(off))
    curved = cv.curve_id[ids] >= 0
    t, e = ring[ts[curved]][:300], ids[curved][:300]
    val, sub, lv = ev.near_pairs(t, e)
    ref = np.array([O.near_pair(x, y, k) for (x, y), k in zip(t, e)])
    scale = np.abs(ref[:, 1]).max()
    assert np.abs(val - ref[:, 0]).max() <= 1e-12 * scale
    assert np.abs(sub - ref[:, 1]).max() <= 1e-13 * scale
    assert np.array_equal(lv, ref[:, 2].astype(np.int64))
    keep = (s >= 0) & (cv.curve_id[np.maximum(s, 0)] >= 0)
    t2, e2 = ring[keep], s[keep]
    val, sub, pn = ev.self_pairs(t2, e2)
    ref = np.array([O.self_pair(x, y, k) for (x, y), k in zip(t2, e2)])
    scale = np.abs(ref[:, 1]).max()
    assert np.abs(val - ref[:, 0]).max() <= 1e-12 * scale
    assert np.array_equal(pn, ref[:, 2].astype(np.int64))


def test_curved_disk_constant_density_exact_on_gpu():
    pr = vp.load_config(2)
    tri, cv = vp.curve_boundary_of_disk(pr.vxy, pr.tri)
    r = vp.make_rules(50, eps=1e-12)
    co = const_coeffs(len(tri), pr.p)
    txy = np.concatenate([pr.txy[::3], ring_targets(2000, seed=9)[:-4]])
    txy = txy[np.hypot(txy[:, 0], txy[:, 1]) <= 1.0]
    ev = vp.Evaluator(0)
    ev.set_mesh(pr.vxy, tri)
    ev.set_curves(cv)
    ev.set_rules(r)
    ev.set_density(pr.p, co)
    u, st = ev.evaluate(txy)
    exact = (np.sum(txy ** 2, 1) - 1) / 4
    assert np.abs(u - exact).max() < 5e-12
    assert st["n_outside"] == 0
    # without the curves the polygon misses the boundary layer
    ev.set_curves(None)
    ev.set_rules(r)
    us, st2 = ev.evaluate(txy)
    assert np.abs(us - exact).max() > 1e-10
    ev.close()


def test_curved_ball_model_matches_oracle(disk):
    pr, tri, cv, coeffs, txy, _, _ = disk
    ev = make(pr, coeffs, tri, cv, near_model="ball")
    O = Oracle(pr.vxy, tri, pr.p, coeffs, pr.rules, near_model=1, curves=cv)
    sub = txy[-4000:][::13]
    s_g, off_g, ids_g = ev.build_nearlist(sub)
    s_o, off_o, ids_o = O.nearlist(sub)
    assert np.array_equal(s_g, s_o) and np.array_equal(ids_g, ids_o)
    u_g, st = ev.evaluate(sub)
    u_o, _, sto = O.evaluate(sub)
    assert rel(u_g, u_o) <= REL_TOL
    assert st["n_leaves"] == sto["n_leaves"] and st["n_panels"] == sto["n_panels"]
    ev.close()


def test_curved_fmm_matches_direct(disk):
    pr, tri, cv, coeffs, txy, ev, O = disk
    sub = txy[::3]
    u_d, _ = ev.evaluate(sub)
    ev.set_far_method("fmm")
    u_f, _ = ev.evaluate(sub)
    ev.set_far_method("direct")
    assert rel(u_f, u_d) <= 1e-13


def test_set_curves_usage_errors(disk):
    pr, tri, cv, coeffs, txy, _, _ = disk
    with vp.Evaluator(0) as ev:
        ev.set_mesh(pr.vxy, tri)
        bad = vp.Curves(np.full(len(tri), 9999, dtype=np.int32), cv.deg, cv.cx, cv.cy, cv.length)
        with pytest.raises(vp.VolpotError):
            ev.set_curves(bad)
        bad = vp.Curves(cv.curve_id, cv.deg, cv.cx, cv.cy, -cv.length)
        with pytest.raises(vp.VolpotError):
            ev.set_curves(bad)


def test_ellipse_domain_on_gpu_matches_oracle_and_exact():
    """Arc-length ellipse boundary (BoundaryCurve + annotate_boundary):
    GPU vs oracle (lists, counts, u) and f = 1 against the closed form."""
    from scipy.integrate import quad
    a, b = 2.0, 1.0
    pr = vp.load_config(2)
    E = vp.BoundaryCurve.ellipse(a, b)
    meta, vxy = vp.annotate_boundary(pr.vxy * np.array([a, b]), pr.tri, [E])
    tri, cv = vp.curves_from_annotation(vxy, pr.tri, meta, [E])
    r = vp.make_rules(50, eps=1e-12)
    co = const_coeffs(len(tri), pr.p)
    ev = vp.Evaluator(0)
    ev.set_mesh(vxy, tri)
    ev.set_curves(cv)
    ev.set_rules(r)
    ev.set_density(pr.p, co)
    s_ = np.linspace(0, E.length, 3001)[:-1]
    bpts = E.points(s_)[0] * (1 - np.linspace(0, 1e-3, s_.size))[:, None]
    txy = np.concatenate([pr.txy * np.array([a, b]), bpts])
    u, st = ev.evaluate(txy)
    R = lambda th: a * b / np.sqrt((b * np.cos(th)) ** 2 + (a * np.sin(th)) ** 2)
    C0 = sum(quad(lambda th: R(th) ** 2 / 2 * np.log(R(th)) - R(th) ** 2 / 4, k * np.pi / 4, (k + 1) * np.pi / 4,
                  epsabs=1e-16, epsrel=1e-16)[0] for k in range(8)) / (2 * np.pi)
    exact = C0 + (b * txy[:, 0] ** 2 + a * txy[:, 1] ** 2) / (2 * (a + b))
    assert np.abs(u - exact).max() <= 5e-12
    assert st["n_outside"] == 0
    O = Oracle(vxy, tri, pr.p, co, r, curves=cv)
    sub = np.concatenate([txy[:-3000][::211], bpts[::5]])
    s_g, off_g, ids_g = ev.build_nearlist(sub)
    s_o, off_o, ids_o = O.nearlist(sub)
    assert np.array_equal(s_g, s_o) and np.array_equal(ids_g, ids_o)
    u_g, st_g = ev.evaluate(sub)
    u_o, _, st_o = O.evaluate(sub)
    assert rel(u_g, u_o) <= REL_TOL
    for k in ("n_leaves", "n_panels", "n_degenerate", "n_rho_le1"):
        assert st_g[k] == st_o[k], k
    ev.close()
