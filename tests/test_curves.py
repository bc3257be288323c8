"""Boundary curves and curved-element setup, CPU only.

Mirrors the reference's own curve tests (proj/tests/test_boundary.cpp:40-105:
circle length and point, ellipse length against an adaptive integral,
unit speed, Hermite samples, non-closed rejection), pins the arc-length
parametrisation against the reference's ArcLengthCurve compiled from
/root/reference (oracle/_ref), and checks annotate_boundary's invariants
 and an exact potential on an elliptic domain."""
import io

import numpy as np
import pytest
from scipy.integrate import quad

import paper_2205_04401_b200 as vp
from helpers import const_coeffs
from oracle import binding
from oracle.binding import Oracle

TWO_PI = 2 * np.pi
pytestmark = pytest.mark.filterwarnings("ignore::scipy.integrate.IntegrationWarning")


def herm_circle(n=64):
    t = np.arange(n) / n
    a = TWO_PI * t
    return np.stack([t, np.cos(a), np.sin(a), -TWO_PI * np.sin(a), TWO_PI * np.cos(a)], 1)


def test_unit_circle_length_point_and_closure():
    c = vp.BoundaryCurve.circle()
    assert abs(c.length - TWO_PI) <= 1e-12
    assert c.ccw
    q = c.points(c.length / 4)[0][0]
    assert abs(q[0]) <= 1e-15 and abs(q[1] - 1.0) <= 1e-15
    p0, pl = c.points([0.0, c.length])[0]
    assert np.hypot(*(p0 - pl)) <= 1e-12 * c.length


def test_ellipse_length_matches_adaptive_integral():
    c = vp.BoundaryCurve.ellipse(2.0, 1.0)
    sp = lambda t: np.hypot(2.0 * TWO_PI * np.sin(TWO_PI * t), TWO_PI * np.cos(TWO_PI * t))
    ref = sum(quad(sp, k / 8, (k + 1) / 8, epsabs=1e-15, epsrel=1e-15)[0] for k in range(8))
    assert abs(c.length - ref) <= 1e-12


@pytest.mark.parametrize("make", [lambda: vp.BoundaryCurve.circle(), lambda: vp.BoundaryCurve.ellipse(2.0, 1.0),
                                  lambda: vp.BoundaryCurve.wobbly(1.0, 0.15, 7)])
def test_unit_speed_parametrisation(make):
    c = make()
    L = c.length
    s = L * (np.arange(64) + 0.37) / 64
    _, tg, dd = c.points(s)
    assert np.abs(np.hypot(tg[:, 0], tg[:, 1]) - 1).max() <= 1e-14
    h = 1e-6 * L
    fd = (c.points(s + h)[0] - c.points(s - h)[0]) / (2 * h)
    assert np.abs(fd - tg).max() < 1e-6
    assert np.abs(np.sum(tg * dd, 1)).max() < 1e-12


def test_wobbly_inverse_is_exact_against_high_precision_integral():
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 30
    a, b, k = 1.0, 0.15, 7
    c = vp.BoundaryCurve.wobbly(a, b, k)

    def speed(t):
        u = 2 * mp.pi * t
        r, rp = a + b * mp.cos(k * u), -b * k * mp.sin(k * u)
        return 2 * mp.pi * mp.sqrt(rp ** 2 + r ** 2)

    for t in (0.37, 0.811):
        s = mp.quad(speed, list(mp.linspace(0, t, 60)))
        assert abs(c.param(float(s)) - t) <= 1e-15


def test_hermite_samples_reproduce_a_circle():
    text = "# t x y dx dy\n" + "\n".join(" ".join(f"{v:.17g}" for v in row) for row in herm_circle())
    from paper_2205_04401_b200 import formats
    rows = formats.read_curve_samples(io.StringIO(text))
    c = vp.BoundaryCurve.hermite(rows)
    assert abs(c.length - TWO_PI) <= 1e-6
    assert abs(np.hypot(*c.points(0.3 * c.length)[0][0]) - 1.0) <= 1e-7


def test_curve_usage_errors():
    with pytest.raises(vp.VolpotError, match="not closed"):
        vp.BoundaryCurve.arc(0.0, 0.0, 1.0, 0.0, 3.0)
    with pytest.raises(vp.VolpotError, match="a > \\|b\\|"):
        vp.BoundaryCurve.wobbly(0.1, 0.2, 3)
    bad = herm_circle()
    bad[3, 0] = bad[2, 0]
    with pytest.raises(vp.VolpotError, match="increase"):
        vp.BoundaryCurve.hermite(bad)
    with pytest.raises(vp.VolpotError, match="3 consistent"):
        vp.BoundaryCurve.hermite(herm_circle()[:2])


REF_CASES = [
    (0, [0.3, -0.2, 1.7], lambda: vp.BoundaryCurve.circle(0.3, -0.2, 1.7), 1e-12),
    (1, [2.0, 1.0], lambda: vp.BoundaryCurve.ellipse(2.0, 1.0), 1e-12),
    # the reference interpolates t(s) by 64 x order-16 Chebyshev panels; on
    # the k = 7 wobble that interpolant carries ~2e-10 (ours is exact, above)
    (2, [1.0, 0.15, 7], lambda: vp.BoundaryCurve.wobbly(1.0, 0.15, 7), 1e-9),
    (3, herm_circle(), lambda: vp.BoundaryCurve.hermite(herm_circle()), 1e-12),
]


@pytest.mark.parametrize("kind,prm,make,tol", REF_CASES)
def test_arc_length_pinned_against_reference(kind, prm, make, tol):
    if binding.ref() is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    c = make()
    s = np.linspace(0, c.length, 401)[:-1] + 0.0123
    xr, tr, dr, Lr, ccw = binding.ref_arclength(kind, prm, s)
    x, tg, dd = c.points(s)
    assert abs(c.length - Lr) <= 1e-12 * Lr
    assert ccw == c.ccw
    assert np.abs(x - xr).max() <= tol
    assert np.abs(tg - tr).max() <= 10 * tol


def test_segment_series_reproduces_the_curve():
    c = vp.BoundaryCurve.ellipse(2.0, 1.0)
    sa, sb = 1.1, 1.25
    from numpy.polynomial import legendre as L
    for s_from, s_to in ((sb, sa), (sa, sb)):
        gx, gy, ln = c.segment(s_from, s_to, 16)
        assert abs(ln - 0.15) <= 1e-15
        tau = np.linspace(0, 1, 23)
        ref = c.points(s_from + tau * (s_to - s_from))[0]
        assert np.abs(L.legval(2 * tau - 1, gx) - ref[:, 0]).max() <= 1e-14
        assert np.abs(L.legval(2 * tau - 1, gy) - ref[:, 1]).max() <= 1e-14


def test_annotate_boundary_invariants_on_the_disk(tmp_path):
    pr = vp.load_config(2)
    C = vp.BoundaryCurve.circle()
    meta, vxy = vp.annotate_boundary(pr.vxy, pr.tri, [C])
    curved = meta[:, 0] != 0
    assert curved.sum() == 256  # = boundary edges
    cover = np.sum((meta[curved, 4] - meta[curved, 3]) % C.length)
    assert abs(cover - C.length) <= 1e-8
    tri, cv = vp.curves_from_annotation(vxy, pr.tri, meta, [C])
    tri0, cv0 = vp.curve_boundary_of_disk(pr.vxy, pr.tri)
    assert np.array_equal(tri, tri0) and np.array_equal(cv.curve_id, cv0.curve_id)
    assert np.abs(cv.cx - cv0.cx).max() <= 1e-15 and np.abs(cv.cy - cv0.cy).max() <= 1e-15
    # endpoints: G(0) = v1, G(1) = v0 (the element's (gamma(L), gamma(0), O) order)
    from numpy.polynomial import legendre as L
    e = np.nonzero(cv.curve_id >= 0)[0]
    g0 = np.stack([L.legval(-1.0, cv.cx[cv.curve_id[e]].T), L.legval(-1.0, cv.cy[cv.curve_id[e]].T)], 1)
    g1 = np.stack([L.legval(1.0, cv.cx[cv.curve_id[e]].T), L.legval(1.0, cv.cy[cv.curve_id[e]].T)], 1)
    assert np.abs(g0 - vxy[tri[e, 1]]).max() <= 1e-14 and np.abs(g1 - vxy[tri[e, 0]]).max() <= 1e-14
    # mesh file round trip with the curved annotation
    from paper_2205_04401_b200 import formats
    path = tmp_path / "disk.mesh"
    formats.write_mesh(path, vxy, pr.tri, meta=meta)
    v2, t2, _, m2 = formats.read_mesh(path, with_meta=True)
    assert np.array_equal(v2, vxy) and np.array_equal(t2, pr.tri) and np.array_equal(m2, meta)
    with pytest.raises(ValueError, match="with_meta"):
        formats.read_mesh(path)


def test_ellipse_domain_constant_density_is_exact():
    """f = 1 on the ellipse x^2/a^2 + y^2/b^2 <= 1: u = C0 + (b x^2 + a y^2)/(2(a+b))
    with C0 = (1/2pi) int_0^2pi (R^2/2 log R - R^2/4) dtheta.  The disk mesh
    stretched to the ellipse, its boundary elements blended onto the exact
    ellipse (annotate_boundary + curves_from_annotation)."""
    a, b = 2.0, 1.0
    pr = vp.load_config(2)
    E = vp.BoundaryCurve.ellipse(a, b)
    meta, vxy = vp.annotate_boundary(pr.vxy * np.array([a, b]), pr.tri, [E])
    tri, cv = vp.curves_from_annotation(vxy, pr.tri, meta, [E])
    R = lambda th: a * b / np.sqrt((b * np.cos(th)) ** 2 + (a * np.sin(th)) ** 2)
    C0 = sum(quad(lambda th: R(th) ** 2 / 2 * np.log(R(th)) - R(th) ** 2 / 4, k * np.pi / 4, (k + 1) * np.pi / 4,
                  epsabs=1e-16, epsrel=1e-16)[0] for k in range(8)) / TWO_PI
    th = np.linspace(0.1, 6.0, 7)
    txy = np.concatenate([(pr.txy * np.array([a, b]))[::1231], np.stack([a * np.cos(th), b * np.sin(th)], 1)])
    exact = C0 + (b * txy[:, 0] ** 2 + a * txy[:, 1] ** 2) / (2 * (a + b))
    u, _, _ = Oracle(vxy, tri, pr.p, const_coeffs(len(tri), pr.p), vp.make_rules(50, eps=1e-12),
                     curves=cv).evaluate(txy)
    assert np.abs(u - exact).max() <= 5e-12
