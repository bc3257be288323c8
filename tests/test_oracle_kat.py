"""Known-answer tests of the CPU oracle's hot path (independent of the GPU).

The reference pins nothing on this path, so the oracle is
checked against closed forms and independent quadrature instead:
  * f = 1: the potential of a triangle has a closed form (divergence theorem);
  * f linear: scipy adaptive quadrature in polar coordinates about the target;
  * the SPEC's examples for far/near/self."""
import numpy as np
import pytest
from scipy import integrate

import paper_2205_04401_b200 as vp
from helpers import brute_nearlist, const_coeffs, small_mesh, tri_potential_const
from oracle.binding import Oracle


@pytest.fixture(scope="module")
def cfg1():
    return vp.load_config(1)


@pytest.mark.parametrize("eps,tol", [(1e-8, 5e-8), (1e-10, 5e-10), (1e-12, 5e-12), (1e-14, 2e-13)])
def test_constant_density_matches_closed_form(cfg1, eps, tol):
    """SPEC acceptance 1 analogue: |u - exact| <= tol for f = 1 at every eps."""
    pr = cfg1
    O = Oracle(pr.vxy, pr.tri, pr.p, const_coeffs(pr.n_tri, pr.p), vp.make_rules(pr.q, eps=eps))
    u, _, st = O.evaluate(pr.txy)
    ua = tri_potential_const(pr.vxy, pr.tri, pr.txy)
    assert np.abs(u - ua).max() <= tol


def test_counts_shrink_with_eps_and_q(cfg1):
    """c and s_n are monotone in eps (SPEC nearfield monotonicity) and in q
    (offloading)."""
    pr = cfg1
    sub = pr.txy[::7]
    prev = None
    for eps in (1e-14, 1e-12, 1e-10, 1e-8):
        O = Oracle(pr.vxy, pr.tri, pr.p, pr.coeffs, vp.make_rules(pr.q, eps=eps))
        _, _, st = O.evaluate(sub)
        if prev:
            assert st["n_near_pairs"] <= prev["n_near_pairs"] and st["n_leaves"] <= prev["n_leaves"]
        prev = st
    prev = None
    for q in (6, 10, 16, 24):
        O = Oracle(pr.vxy, pr.tri, pr.p, pr.coeffs, vp.make_rules(q))
        s, off, ids = O.nearlist(sub)
        if prev is not None:
            assert len(ids) <= prev
        prev = len(ids)


def _poly_integral_polar(vxy, tri_idx, t, f):
    """(1/2pi) int_T log|t-y| f(y) dA by scipy dblquad in polar coordinates
    about t over the three sub-triangles (t, A, B) (smooth integrands)."""
    P = vxy[tri_idx]
    tot = 0.0
    for k in range(3):
        A, B = P[k], P[(k + 1) % 3]

        def rmax(th, A=A, B=B):
            d = np.array([np.cos(th), np.sin(th)])
            M = np.array([d, A - B]).T
            sol = np.linalg.solve(M, A - t)
            return sol[0]
        a0 = np.arctan2(*(A - t)[::-1])
        a1 = np.arctan2(*(B - t)[::-1])
        if a1 < a0:
            a1 += 2 * np.pi
        val, _ = integrate.dblquad(
            lambda r, th: np.log(r) * f(t[0] + r * np.cos(th), t[1] + r * np.sin(th)) * r,
            a0, a1, 0.0, rmax, epsabs=1e-15, epsrel=1e-13)
        tot += val
    return tot / (2 * np.pi)


def _outside_integral(vxy, tri_idx, t, f):
    P = vxy[tri_idx]
    x0, e1, e2 = P[0], P[1] - P[0], P[2] - P[0]
    det = e1[0] * e2[1] - e2[0] * e1[1]

    def g(eta, xi):
        y = x0 + xi * e1 + eta * e2
        return np.log(np.hypot(*(t - y))) * f(*y) * det
    val, _ = integrate.dblquad(g, 0, 1, 0, lambda xi: 1 - xi, epsabs=1e-15, epsrel=1e-13)
    return val / (2 * np.pi)


def test_self_eval_linear_density_against_adaptive_quadrature():
    """self_eval vs an adaptive polar oracle (SPEC.md:517-526 example class)."""
    vxy = np.array([[0.0, 0.0], [1.0, 0.1], [0.3, 0.8]])
    tri = np.array([[0, 1, 2]], dtype=np.int32)
    a, b, c = 0.7, -0.4, 1.3
    p = 2
    co = vp.project_density(vxy, tri, p, vp.F_LINEAR, [a, b, c])
    O = Oracle(vxy, tri, p, co, vp.make_rules(6))
    f = lambda x, y: a + b * x + c * y  # noqa: E731
    for t in ([0.4, 0.3], [0.45, 0.32], [0.05, 0.02], [0.9, 0.1]):
        t = np.array(t)
        val, _, panels = O.self_pair(t[0], t[1], 0)
        ref = _poly_integral_polar(vxy, tri[0], t, f)
        assert abs(val - ref) <= 1e-12, (t, val, ref)
        assert panels >= 6


def test_near_eval_linear_density_against_adaptive_quadrature():
    vxy = np.array([[0.0, 0.0], [1.0, 0.1], [0.3, 0.8]])
    tri = np.array([[0, 1, 2]], dtype=np.int32)
    a, b, c = 0.7, -0.4, 1.3
    co = vp.project_density(vxy, tri, 2, vp.F_LINEAR, [a, b, c])
    O = Oracle(vxy, tri, 2, co, vp.make_rules(16))
    f = lambda x, y: a + b * x + c * y  # noqa: E731
    for t in ([0.5, -0.01], [0.5, -0.2], [1.05, 0.1], [-0.3, -0.3]):
        t = np.array(t)
        val, sub, leaves, depth = O.near_pair(t[0], t[1], 0)
        ref = _outside_integral(vxy, tri[0], t, f)
        assert abs(val - ref) <= 1e-12, (t, val, ref)


def test_near_eval_far_away_is_one_leaf():
    """a far target needs zero subdivisions."""
    vxy, tri = small_mesh()
    co = const_coeffs(2, 2)
    O = Oracle(vxy, tri, 2, co, vp.make_rules(16))
    val, sub, leaves, depth = O.near_pair(30.0, -20.0, 0)
    assert leaves == 1 and depth == 0
    assert abs(val - sub) <= 1e-15 * abs(sub) * 10


def test_far_sum_of_zero_density_is_zero(cfg1):
    pr = cfg1
    O = Oracle(pr.vxy, pr.tri, pr.p, np.zeros_like(pr.coeffs), pr.rules)
    assert np.all(O.far_sum(pr.txy[:100]) == 0.0)


def test_isometry_invariance(cfg1):
    """Rotation + translation invariance of the full evaluation (SPEC quadrature-engine)."""
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.1, 0.9], [1.1, 1.0]])
    tri = np.array([[0, 1, 3], [0, 3, 2]], dtype=np.int32)
    p = 3
    co = vp.project_density(vxy, tri, p, vp.F_LINEAR, [1.0, 0.5, -0.25])
    lx, ly = vp.lattice_nodes(p)
    txy = np.concatenate([vxy[t[0]] + np.outer(lx, vxy[t[1]] - vxy[t[0]]) + np.outer(ly, vxy[t[2]] - vxy[t[0]])
                          for t in tri])
    txy = np.vstack([txy, [[1.3, 0.4], [-0.2, 0.5]]])
    r = vp.make_rules(10)
    u0, _, _ = Oracle(vxy, tri, p, co, r).evaluate(txy)
    th = 0.7
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    sh = np.array([3.0, -2.0])
    # the density is attached to the elements, so coefficients are unchanged
    u1, _, _ = Oracle(vxy @ R.T + sh, tri, p, co, r).evaluate(txy @ R.T + sh)
    assert np.abs(u0 - u1).max() <= 1e-13


def test_lists_match_brute_force_scan(cfg1):
    pr = cfg1
    O = Oracle.from_problem(pr)
    rho0, rho0n, ta = O.element_models()
    sub = pr.txy[::5]
    s, off, ids = O.nearlist(sub)
    sb, offb, idsb = brute_nearlist(pr.vxy, pr.tri, ta, rho0 <= 1.0, sub)
    assert np.array_equal(s, sb) and np.array_equal(off, offb) and np.array_equal(ids, idsb)


def test_targets_outside_and_on_boundaries():
    vxy, tri = small_mesh()
    p = 2
    co = const_coeffs(2, p)
    O = Oracle(vxy, tri, p, co, vp.make_rules(10))
    txy = np.array([[2.0, 2.0], [-0.5, 0.5], [0.5, 0.5], [0.0, 0.0], [1.0, 0.0], [0.25, 0.0], [0.3, 0.3]])
    s, off, ids = O.nearlist(txy)
    assert s[0] == -1 and s[1] == -1
    assert s[2] == 0  # on the shared diagonal: lowest id
    assert s[3] == 0 and s[4] == 0 and s[5] == 0
    u, _, st = O.evaluate(txy)
    ua = tri_potential_const(vxy, tri, txy)
    # targets on a side of a neighbour are handled at the eps level
    assert np.abs(u - ua).max() <= 5e-12
    assert st["n_outside"] == 2


def test_all_near_elements_when_rho0_le_1():
    """eps so large that rho0 <= 1: every element is all-near."""
    vxy, tri = small_mesh()
    co = const_coeffs(2, 1)
    O = Oracle(vxy, tri, 1, co, vp.make_rules(6, eps=1.0))
    rho0, _, _ = O.element_models()
    assert (rho0 <= 1).all()
    s, off, ids = O.nearlist(np.array([[5.0, 5.0], [0.2, 0.1]]))
    assert list(ids[off[0]:off[1]]) == [0, 1] and list(ids[off[1]:off[2]]) == [1]


def test_empty_target_array(cfg1):
    O = Oracle.from_problem(cfg1)
    s, off, ids = O.nearlist(np.zeros((0, 2)))
    assert len(s) == 0 and list(off) == [0] and len(ids) == 0
    u, _, st = O.evaluate(np.zeros((0, 2)))
    assert len(u) == 0


def test_ball_model_lists_match_brute_force_and_is_coarser_on_the_disk():
    """Ball baseline: lists equal a brute-force scan, and on the
    disk the precise model needs fewer corrections (PAPER.md Table near_corr)."""
    pr = vp.load_config(2)
    sub = pr.txy[::509]
    Ob = Oracle.from_problem(pr, near_model=1)
    s, off, ids = Ob.nearlist(sub)
    P = pr.vxy[pr.tri]
    a, b, c = P[:, 0], P[:, 1], P[:, 2]
    bxr, byr, cxr, cyr = b[:, 0] - a[:, 0], b[:, 1] - a[:, 1], c[:, 0] - a[:, 0], c[:, 1] - a[:, 1]
    d = 2.0 * (bxr * cyr - byr * cxr)
    b2, c2 = bxr * bxr + byr * byr, cxr * cxr + cyr * cyr
    ux, uy = (cyr * b2 - byr * c2) / d, (bxr * c2 - cxr * b2) / d
    rr = 2.25 * (ux * ux + uy * uy)
    for k, t in enumerate(sub):
        dx, dy = (t[0] - a[:, 0]) - ux, (t[1] - a[:, 1]) - uy
        near = set(np.nonzero(dx * dx + dy * dy < rr)[0]) - {s[k]}
        assert sorted(near) == list(ids[off[k]:off[k + 1]])
    _, _, stb = Ob.evaluate(sub)
    _, _, stp = Oracle.from_problem(pr).evaluate(sub)
    assert stp["n_near_pairs"] < stb["n_near_pairs"] and stp["n_leaves"] < stb["n_leaves"]


# ---------------------------------------------------------------------------
# curved (blending-map) elements, SURVEY.md §8(f3)

def _disk_sample(stride=617):
    pr = vp.load_config(2)
    return pr, pr.txy[::stride]


def test_circle_arc_coefficients_reproduce_the_arc():
    gx, gy, ln = vp.circle_arc(0.5, -0.25, 2.0, 0.3, 0.1, deg=16)
    assert abs(ln - 0.4) < 1e-15
    tau = np.linspace(0, 1, 41)
    from numpy.polynomial import legendre as L
    x, y = L.legval(2 * tau - 1, gx), L.legval(2 * tau - 1, gy)
    th = 0.3 + tau * (0.1 - 0.3)
    assert np.abs(x - (0.5 + 2 * np.cos(th))).max() < 1e-15
    assert np.abs(y - (-0.25 + 2 * np.sin(th))).max() < 1e-15


def test_curved_disk_constant_density_is_exact():
    """f = 1 on the exact unit disk: u = (|x|^2 - 1)/4.  The polygonal mesh
    misses it by its O(h^2) domain error; blended boundary elements reach eps."""
    pr, sub = _disk_sample()
    th = np.linspace(0.1, 6.0, 13)  # targets on the arcs themselves
    sub = np.concatenate([sub, np.stack([np.cos(th), np.sin(th)], 1)])
    tri, cv = vp.curve_boundary_of_disk(pr.vxy, pr.tri)
    assert (cv.curve_id >= 0).sum() == 256
    co = const_coeffs(len(tri), pr.p)
    r = vp.make_rules(50, eps=1e-12)
    exact = (np.sum(sub ** 2, 1) - 1) / 4
    u, _, _ = Oracle(pr.vxy, tri, pr.p, co, r, curves=cv).evaluate(sub)
    us, _, _ = Oracle(pr.vxy, tri, pr.p, co, r).evaluate(sub)
    assert np.abs(u - exact).max() < 5e-12
    assert np.abs(us - exact).max() > 1e-10


def test_curved_element_with_straight_side_equals_straight_element():
    """A blending map over a straight gamma is the affine map, so marking an
    element curved with its chord as gamma must not change u."""
    pr, sub = _disk_sample(stride=1201)
    tri, cv = vp.curve_boundary_of_disk(pr.vxy, pr.tri)
    chord = np.zeros_like(cv.cx), np.zeros_like(cv.cy)
    for e in np.nonzero(cv.curve_id >= 0)[0]:
        c = cv.curve_id[e]
        a, b = pr.vxy[tri[e, 0]], pr.vxy[tri[e, 1]]  # gamma(L) = a, gamma(0) = b
        chord[0][c, 0], chord[0][c, 1] = (a[0] + b[0]) / 2, (a[0] - b[0]) / 2
        chord[1][c, 0], chord[1][c, 1] = (a[1] + b[1]) / 2, (a[1] - b[1]) / 2
    flat = vp.Curves(cv.curve_id, cv.deg, chord[0], chord[1], np.hypot(chord[0][:, 1], chord[1][:, 1]) * 2)
    r = vp.make_rules(50, eps=1e-12)
    co = vp.project_density(pr.vxy, tri, pr.p, vp.F_GAUSS, [0.2, -0.1, 3.0])
    u1, _, _ = Oracle(pr.vxy, tri, pr.p, co, r, curves=flat).evaluate(sub)
    u0, _, _ = Oracle(pr.vxy, tri, pr.p, co, r).evaluate(sub)
    assert np.abs(u1 - u0).max() < 1e-12 * max(1.0, np.abs(u0).max())
