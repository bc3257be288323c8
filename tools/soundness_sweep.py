"""Near-field soundness sweep (SPEC.md:458, :754 acceptance criterion 4;
PAPER.md Figs. nf0/nf1/nf2) with this repo's substitute far rules.

For a triangle T, a far rule of order q (collapsed Gauss-Jacobi, the rules
both the oracle and the GPU use), a density f and a tolerance eps, the
three-ellipse model (rho0 = (w_edge |J| / (eps C_q))^(1/q))
classifies exterior points as near or far.  Soundness: every far point has
|far-rule I_T(x) - I_T(x)| <= eps, with I_T(x) = int_T log|x-y| f(y) dA and
the reference value from the adaptive oracle (oracle/vp_oracle_accept.cpp).

Points: a 50 x 50 grid over the triangle's bbox grown by one diameter,
exterior only (the SPEC's "2000 exterior grid points"), plus 200 points per
side just outside that side's ellipse (rho = 1.001 rho0), where the model is
tightest.

  python tools/soundness_sweep.py [--out profiles/r02_soundness.json]

Used by tests/test_spec_acceptance.py (a reduced sweep) and for the DESIGN
table.  Test infrastructure: uses oracle/ only.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import binding as B  # noqa: E402

F_NAMES = {0: "1", 1: "sin(x+2y)", 2: "exp(-x^2-y^2)", 3: "Koornwinder poly"}


def random_triangles(n, seed=2205, max_aspect=4.0):
    """n random CCW triangles of diameter ~1 with aspect ratio (longest side^2 /
    (2 area)) <= max_aspect (SPEC.md: the model is asserted for aspect <= 4)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        v = rng.uniform(-0.5, 0.5, size=(3, 2)) + rng.uniform(-2, 2, size=2)
        d = (v[1, 0] - v[0, 0]) * (v[2, 1] - v[0, 1]) - (v[2, 0] - v[0, 0]) * (v[1, 1] - v[0, 1])
        if d < 0:
            v = v[[0, 2, 1]]
            d = -d
        L = max(np.sum((v[(k + 1) % 3] - v[k]) ** 2) for k in range(3))
        if d > 1e-3 and L / d <= max_aspect:
            out.append(v.reshape(6))
    return out


def model(tri, q, eps, rule):
    """(rho0, [2a per side]) of the precise model, the oracle's formula."""
    x, y, w = rule
    v = np.asarray(tri).reshape(3, 2)
    det = (v[1, 0] - v[0, 0]) * (v[2, 1] - v[0, 1]) - (v[2, 0] - v[0, 0]) * (v[1, 1] - v[0, 1])
    we = B.w_edge(x, y, w)
    rho0 = (we * det / (eps * B.cn_lookup(q))) ** (1.0 / q)
    lens = [np.hypot(*(v[(k + 1) % 3] - v[k])) for k in range(3)]
    return rho0, [0.5 * (rho0 + 1 / rho0) * L for L in lens]


def classify(tri, pts, rho0, two_a):
    """0 far, 1 near (inside an open ellipse, or rho0 <= 1: all-near)."""
    v = np.asarray(tri).reshape(3, 2)
    if rho0 <= 1.0:
        return np.ones(len(pts), dtype=bool)
    d = [np.hypot(pts[:, 0] - v[k, 0], pts[:, 1] - v[k, 1]) for k in range(3)]
    return (d[0] + d[1] < two_a[0]) | (d[1] + d[2] < two_a[1]) | (d[2] + d[0] < two_a[2])


def inside(tri, pts, tol=1e-12):
    v = np.asarray(tri).reshape(3, 2)
    e1, e2 = v[1] - v[0], v[2] - v[0]
    det = e1[0] * e2[1] - e2[0] * e1[1]
    d = pts - v[0]
    xi = (e2[1] * d[:, 0] - e2[0] * d[:, 1]) / det
    eta = (-e1[1] * d[:, 0] + e1[0] * d[:, 1]) / det
    return (xi >= -tol) & (eta >= -tol) & (1 - xi - eta >= -tol)


def ellipse_shell(tri, rho0, two_a, n=200, grow=1.001):
    """Points on the Bernstein ellipse of parameter grow*rho0 about each side."""
    v = np.asarray(tri).reshape(3, 2)
    out = []
    for k in range(3):
        P, Q = v[k], v[(k + 1) % 3]
        c = 0.5 * np.hypot(*(Q - P))
        r = rho0 * grow
        a, b = c * 0.5 * (r + 1 / r), c * 0.5 * (r - 1 / r)
        u = (Q - P) / (2 * c)
        nv = np.array([-u[1], u[0]])
        th = np.linspace(0, 2 * np.pi, n, endpoint=False) + 0.5 / n
        m = 0.5 * (P + Q)
        out.append(m + np.outer(a * np.cos(th), u) + np.outer(b * np.sin(th), nv))
    return np.concatenate(out)


def grid_points(tri, n=50):
    v = np.asarray(tri).reshape(3, 2)
    lo, hi = v.min(0), v.max(0)
    dm = max(hi - lo)
    g = np.linspace(0, 1, n)
    X, Y = np.meshgrid(lo[0] - dm + g * (hi[0] - lo[0] + 2 * dm), lo[1] - dm + g * (hi[1] - lo[1] + 2 * dm))
    pts = np.stack([X.ravel(), Y.ravel()], 1)
    return pts[~inside(tri, pts)]


def rule_values(tri, pts, rule, fkind, coeffs=None, p=0):
    x, y, w = rule
    v = np.asarray(tri).reshape(3, 2)
    e1, e2 = v[1] - v[0], v[2] - v[0]
    det = e1[0] * e2[1] - e2[0] * e1[1]
    X = v[0, 0] + x * e1[0] + y * e2[0]
    Y = v[0, 1] + x * e1[1] + y * e2[1]
    if fkind == 0:
        f = np.ones_like(X)
    elif fkind == 1:
        f = np.sin(X + 2 * Y)
    elif fkind == 2:
        f = np.exp(-X * X - Y * Y)
    else:
        f = np.array([np.dot(coeffs, B.koornwinder(p, a, b)) for a, b in zip(x, y)])
    r = np.hypot(pts[:, 0:1] - X[None], pts[:, 1:2] - Y[None])
    return (np.log(r) * (w * f)[None]).sum(1) * det


def sweep(tris, fkinds, qs, epss, coeffs=None, p=0, n_grid=50, n_shell=200, nthreads=0):
    """Rows: (tri index, f, q, eps, n far, n far with error > eps, max err/eps over far)."""
    rows = []
    for ti, tri in enumerate(tris):
        for fk in fkinds:
            for q in qs:
                rule = B.quad_rule(q)  # the evaluation's far rule (symmetric where tabulated)
                for eps in epss:
                    rho0, ta = model(tri, q, eps, rule)
                    pts = grid_points(tri, n_grid)
                    if rho0 > 1.0:
                        sh = ellipse_shell(tri, rho0, ta, n_shell)
                        pts = np.concatenate([pts, sh[~inside(tri, sh)]])
                    far = ~classify(tri, pts, rho0, ta)
                    if not far.any():
                        rows.append((ti, fk, q, eps, 0, 0, 0.0, rho0))
                        continue
                    P = pts[far]
                    ex = B.adaptive_log_integral(tri, fk, P, coeffs=coeffs, p=p, nthreads=nthreads)
                    err = np.abs(rule_values(tri, P, rule, fk, coeffs, p) - ex)
                    rows.append((ti, fk, q, eps, int(far.sum()), int((err > eps).sum()), float(err.max() / eps), rho0))
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    tris = [np.array([0, 0, 1, 0, 0, 1.0])] + random_triangles(10)
    qs = [6, 10, 12, 16, 20, 24, 40]
    epss = [1e-8, 1e-10, 1e-12, 1e-14]
    rows = sweep(tris, [0, 1, 2], qs, epss)
    doc = {"what": "near-field soundness sweep (SPEC.md:754), substitute collapsed Gauss-Jacobi rules",
           "columns": ["triangle", "f", "q", "eps", "n_far", "n_fail", "max_err_over_eps", "rho0"],
           "rows": rows}
    # summary per (f, q)
    for fk in (0, 1, 2):
        for q in qs:
            r = [x for x in rows if x[1] == fk and x[2] == q]
            print(f"f={F_NAMES[fk]:14s} q={q:2d}: far {sum(x[4] for x in r):7d} fail {sum(x[5] for x in r):6d} "
                  f"max err/eps {max(x[6] for x in r):9.3g}")
    if a.out:
        json.dump(doc, open(a.out, "w"), indent=0)


if __name__ == "__main__":
    main()
