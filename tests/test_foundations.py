"""Oracle foundations pinned against the reference (CPU).

Mirrors the reference's own unit tests (proj/tests/test_basis.cpp,
test_quadtree.cpp) and compares with golden fixtures produced by the
reference's headers (tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from oracle import binding as ob

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def product_rule(k):
    """collapsed Gauss product rule, the test oracle of test_basis.cpp:14-29"""
    x, w = ob.gauss_legendre(k)
    u, wu = 0.5 * (x + 1), 0.5 * w
    nodes, weights = [], []
    for i in range(k):
        for j in range(k):
            nodes.append((u[i], u[j] * (1 - u[i])))
            weights.append(wu[i] * wu[j] * (1 - u[i]))
    return np.array(nodes), np.array(weights)


def test_k00_is_sqrt2():  # test_basis.cpp:33-38
    for x, y in [(0.1, 0.3), (0.0, 0.0), (0.9999, 0.0), (0.3, 0.7)]:
        assert abs(ob.koornwinder(12, x, y)[0] - np.sqrt(2.0)) <= 1e-14


def test_gram_identity_n12():  # test_basis.cpp:40-55
    N = 12
    nodes, w = product_rule(2 * N + 4)
    V = np.array([ob.koornwinder(N, x, y) for x, y in nodes])
    G = (V * w[:, None]).T @ V
    assert np.abs(G - np.eye(V.shape[1])).max() <= 1e-12


def test_low_order_moments_vanish():  # test_basis.cpp:57-68
    nodes, w = product_rule(30)
    for m, n in [(0, 1), (1, 1), (2, 3)]:
        acc = sum(wi * ob.koornwinder(n, x, y)[vp.koorn_index(m, n)] for (x, y), wi in zip(nodes, w))
        assert abs(acc) <= 1e-13


def test_outside_simplex_is_rejected():  # test_basis.cpp:70-75
    with pytest.raises(ob.OracleError):
        ob.koornwinder(5, -1e-6, 0.2)
    with pytest.raises(ob.OracleError):
        ob.koornwinder(5, 0.6, 0.6)
    ob.koornwinder(5, 0.0, 0.0)
    ob.koornwinder(5, 1.0, 0.0)


def test_koornwinder_bitwise_equal_to_reference_golden():
    g = np.load(os.path.join(GOLD, "koorn_ref.npz"))
    for (x, y), ref in zip(g["pts"], g["vals"]):
        assert np.array_equal(ob.koornwinder(int(g["order"]), x, y), ref)


@pytest.mark.skipif(ob.ref() is None, reason="reference shim not built (no /root/reference here)")
def test_koornwinder_bitwise_equal_to_reference_live():
    rng = np.random.default_rng(7)
    for _ in range(200):
        x, y = rng.random(2)
        if x + y > 1:
            x, y = 1 - x, 1 - y
        for order in (4, 8, 12):
            assert np.array_equal(ob.koornwinder(order, x, y), ob.ref_koornwinder(order, x, y))


def test_gauss_legendre_matches_reference_golden():
    g = np.load(os.path.join(GOLD, "gl_ref.npz"))
    for n in g["ns"]:
        x, w = ob.gauss_legendre(int(n))
        assert np.array_equal(x, g[f"x{n}"]) and np.array_equal(w, g[f"w{n}"])
        xp, wp = vp.gauss_legendre(int(n))  # product host copy of the same algorithm
        assert np.array_equal(xp, g[f"x{n}"]) and np.array_equal(wp, g[f"w{n}"])


def test_quadtree_matches_reference_golden_and_linear_scan():  # test_quadtree.cpp:87-112
    g = np.load(os.path.join(GOLD, "quadtree_ref.npz"))
    P = np.random.default_rng(2024).random((10000, 2))
    assert P.sum() == g["pts_sum"]
    for k, r in enumerate(g["rects"]):
        ids, vis = ob.quadtree_query(P, 8, r)
        ref = g["ids"][g["off"][k]:g["off"][k + 1]]
        assert np.array_equal(ids, ref)
        scan = np.nonzero((P[:, 0] >= r[0]) & (P[:, 0] <= r[2]) & (P[:, 1] >= r[1]) & (P[:, 1] <= r[3]))[0]
        assert np.array_equal(ids, scan)
        assert vis == g["visited"][k]


def test_quadtree_edge_cases():  # test_quadtree.cpp:26-85
    with pytest.raises(ob.OracleError):
        ob.quadtree_query(np.zeros((0, 2)), 8, (0, 0, 1, 1))
    P = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    ids, _ = ob.quadtree_query(P, 1, (-1, -1, 2, 2))
    assert list(ids) == [0, 1, 2, 3]
    ids, _ = ob.quadtree_query(P, 1, (5, 5, 6, 6))
    assert len(ids) == 0
    # coincident overflow (test_quadtree.cpp:65-71)
    pts = np.vstack([np.tile([[0.25, 0.75]], (100, 1)), [[0.9, 0.1]]])
    ids, _ = ob.quadtree_query(pts, 4, (0.2, 0.7, 0.3, 0.8))
    assert len(ids) == 100
    # all points coincident: degenerate root box (the reference recurses
    # without end here; the oracle stops at unsplittable boxes)
    same = np.tile([[0.5, 0.5]], (50, 1))
    ids, _ = ob.quadtree_query(same, 4, (0.5, 0.5, 0.5, 0.5))
    assert len(ids) == 50
    with pytest.raises(ob.OracleError):
        ob.quadtree_query(P, 1, (1, 1, 0, 0))


@pytest.mark.parametrize("q,w_edge", [(6, 3.54e-2), (10, 1.21e-2), (12, 1.17e-2), (16, 5.99e-3), (24, 3.36e-3)])
def test_substitute_rules_pass_validate_rule(q, w_edge):  # rules.hpp:60-85
    x, y, w = vp.simplex_rule(q)
    assert len(x) == (q // 2 + 1) ** 2
    ob.validate_rule(q, x, y, w)
    we = ob.w_edge(x, y, w)
    assert abs(we - w_edge) / w_edge < 5e-3
    assert w.max() <= 10 * we  # PAPER.md:1874-1876 premise


@pytest.mark.parametrize("q,npts", [(6, 12), (10, 25), (12, 33)])
def test_symmetric_rules_from_the_moment_fit(q, npts):
    """vps_quad_rule (the evaluation's far / near rule): the repository's own
    fully symmetric rules (tools/make_sym_rules.py) have the point counts of
    the X-G tables the SPEC names, pass the reference's validate_rule
    contract (rules.hpp:60-85: positive weights, interior points, area,
    exactness), integrate every monomial of degree <= q to rounding, and are
    invariant under the six permutations of the barycentric coordinates."""
    import math
    x, y, w = vp.quad_rule(q)
    assert len(x) == npts
    ob.validate_rule(q, x, y, w)
    for a in range(q + 1):
        for b in range(q + 1 - a):
            ex = math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)
            assert abs((w * x ** a * y ** b).sum() - ex) <= 4e-15 * ex
    # not exact one degree up (the rule is not secretly a larger one)
    errs = [abs((w * x ** a * y ** (q + 1 - a)).sum() * math.factorial(q + 3) / (math.factorial(a) * math.factorial(q + 1 - a)) - 1)
            for a in range(q + 2)]
    assert max(errs) > 1e-6
    pts = {(round(a, 13), round(b, 13), round(c, 13)): ww for a, b, c, ww in zip(1 - x - y, x, y, w)}
    for (a, b, c), ww in pts.items():
        for perm in ((a, c, b), (b, a, c), (b, c, a), (c, a, b), (c, b, a)):
            assert perm in pts and pts[perm] == ww
    assert w.max() <= 10 * ob.w_edge(x, y, w)  # PAPER.md:1874-1876 premise


def test_quad_rule_falls_back_to_gauss_jacobi():
    for q in (8, 16, 24, 40):
        a, b = vp.quad_rule(q), vp.simplex_rule(q)
        assert all(np.array_equal(u, v) for u, v in zip(a, b))


def test_validate_rule_rejects_malformed():  # test_basis.cpp:114-128
    x, y, w = vp.simplex_rule(6)
    with pytest.raises(ob.OracleError, match="non-positive weight"):
        ob.validate_rule(6, x, y, np.where(np.arange(len(w)) == 0, -w, w))
    with pytest.raises(ob.OracleError, match="outside the simplex"):
        ob.validate_rule(6, x + 0.9, y, w)
    with pytest.raises(ob.OracleError, match="sum to the simplex area"):
        ob.validate_rule(6, x, y, w * 1.01)
    with pytest.raises(ob.OracleError, match="exactness"):
        ob.validate_rule(12, x, y, w)


def test_ggq_exactness_and_moments():  # test_basis.cpp:175-184, :206-228
    gx, gw = np.polynomial.legendre.leggauss(64)
    for ng in (2, 5, 8):
        r, w, res = vp.build_ggq(ng)
        assert len(r) == ng + 1 and (r > 0).all() and (r < 1).all() and (w > 0).all()
        assert res <= 1e-13
        assert abs((w * r).sum() - 0.5) <= 1e-14
        assert abs((w * r * np.log(r)).sum() + 0.25) <= 1e-14
        for n in range(ng + 1):
            P = np.polynomial.legendre.Legendre.basis(n)
            # exact b_n with 64-pt GL; c_n by dyadic composite toward 0
            rr = 0.5 * (gx + 1)
            b = (0.5 * gw * rr * P(2 * rr - 1)).sum()
            c = 0.0
            for k in range(80):
                hi, lo = 2.0 ** -k, 2.0 ** -(k + 1)
                s = 0.5 * (lo + hi) + 0.5 * (hi - lo) * gx
                c += (0.5 * (hi - lo) * gw * s * np.log(s) * P(2 * s - 1)).sum()
            assert abs((w * r * P(2 * r - 1)).sum() - b) <= 1e-13
            assert abs((w * r * np.log(r) * P(2 * r - 1)).sum() - c) <= 1e-13


def test_ggq8_against_brute_force_composite():  # test_basis.cpp:186-204 (10^5 panels here)
    r, w, _ = vp.build_ggq(8)
    P8 = np.polynomial.legendre.Legendre.basis(8)
    gx, gw = np.polynomial.legendre.leggauss(4)
    panels = 100000
    lo = np.arange(panels) / panels
    hi = (np.arange(panels) + 1) / panels
    acc = 0.0
    for i in range(4):
        s = 0.5 * (lo + hi) + 0.5 * (hi - lo) * gx[i]
        acc += (0.5 * (hi - lo) * gw[i] * s * np.log(s) * P8(2 * s - 1)).sum()
    assert abs((w * r * np.log(r) * P8(2 * r - 1)).sum() - acc) <= 1e-11


def test_reference_embedded_ggq8_table_is_not_a_valid_rule():
    """Finding: the reference's frozen fallback table (ggq.hpp:184-199) fails
    its own check (test_basis.cpp:230-239): sum w r = 0.5116, sum w r log r =
    -0.2434.  We therefore build the rule by moment fitting instead."""
    g = json.load(open(os.path.join(GOLD, "ggq8_ref.json")))
    r, w = np.array(g["r"]), np.array(g["w"])
    assert abs((w * r).sum() - 0.5) > 1e-3
    assert abs((w * r * np.log(r)).sum() + 0.25) > 1e-3


@pytest.mark.parametrize("n,c", [(50, 1.0), (20, 6.8), (45, 1.5), (12, 12.0), (40, 2.0), (60, 1.0),
                                 (16, 9.4), (6, 12.0), (10, 12.0)])
def test_cn_lookup(n, c):  # SPEC.md:436-438 examples; N < 12 clamped
    assert abs(ob.cn_lookup(n) - c) < 1e-15
    assert vp.cn_lookup(n) == ob.cn_lookup(n)
