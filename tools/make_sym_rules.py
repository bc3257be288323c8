"""Fully symmetric quadrature rules on the reference triangle by moment fitting,
computed from scratch (no third-party tables): for degree d the unknowns are
the weights and orbit parameters of n1 centroid + n21 (a, a, 1-2a) orbits +
n111 (a, b, 1-a-b) orbits, the equations the integrals of the S3-invariant
polynomials e2^i e3^j (2i + 3j <= d; e2 = l1 l2 + l2 l3 + l3 l1, e3 = l1 l2 l3),
as many as unknowns.  Levenberg-Marquardt from seeded random starts until a
rule with positive weights and interior points appears, then Newton in
50-digit arithmetic (mpmath) to full double precision.

  python tools/make_sym_rules.py OUT.inc [degree:n1:n21:n111 ...]

writes the orbit tables as a C initialiser list, included by the product's
host setup (csrc/sym_rules.inc) and by the oracle's own generator
(oracle/sym_rules.inc)."""
import math
import sys
from fractions import Fraction as F

import mpmath as mp
import numpy as np
from scipy.optimize import least_squares

DEFAULT = ["6:0:2:1", "10:1:2:3", "12:0:5:3"]


def invariants(deg):
    return [(i, j) for j in range(deg // 3 + 1) for i in range((deg - 3 * j) // 2 + 1)]


def exact_moments(deg):
    """integrals of e2^i e3^j over the triangle (0,0),(1,0),(0,1), as fractions"""
    def mul(f, g):
        h = {}
        for (a, b), c in f.items():
            for (d, e), k in g.items():
                h[(a + d, b + e)] = h.get((a + d, b + e), 0) + c * k
        return h

    def add(f, g):
        h = dict(f)
        for k, c in g.items():
            h[k] = h.get(k, 0) + c
        return h

    def power(f, n):
        r = {(0, 0): F(1)}
        for _ in range(n):
            r = mul(r, f)
        return r
    x, y, l3 = {(1, 0): F(1)}, {(0, 1): F(1)}, {(0, 0): F(1), (1, 0): F(-1), (0, 1): F(-1)}
    e2 = add(add(mul(x, y), mul(y, l3)), mul(l3, x))
    e3 = mul(mul(x, y), l3)
    out = []
    for i, j in invariants(deg):
        f = mul(power(e2, i), power(e3, j))
        out.append(sum(c * F(math.factorial(a) * math.factorial(b), math.factorial(a + b + 2)) for (a, b), c in f.items()))
    return out


def orbit_terms(p, n1, n21, n111, one=1.0):
    """(orbit weight sum, e2, e3) of every orbit for the parameter vector p"""
    k, out = 0, []
    if n1:
        out.append((p[0], one / 3, one / 27))
        k = 1
    for _ in range(n21):
        w, a = p[k], p[k + 1]
        k += 2
        out.append((3 * w, 2 * a - 3 * a * a, a * a * (1 - 2 * a)))
    for _ in range(n111):
        w, a, b = p[k], p[k + 1], p[k + 2]
        k += 3
        c = 1 - a - b
        out.append((6 * w, a * b + (a + b) * c, a * b * c))
    return out


def search(deg, n1, n21, n111, seed=1, max_tries=100000):
    IJ = invariants(deg)
    assert len(IJ) == n1 + 2 * n21 + 3 * n111, "square system: unknowns = S3 invariants up to the degree"
    rhs = np.array([float(m) for m in exact_moments(deg)])
    I, J = np.array([i for i, _ in IJ]), np.array([j for _, j in IJ])

    def res(p):
        t = orbit_terms(p, n1, n21, n111)
        W, E2, E3 = (np.array(v) for v in zip(*t))
        return (W[:, None] * E2[:, None] ** I[None, :] * E3[:, None] ** J[None, :]).sum(0) / rhs - 1.0
    rng = np.random.default_rng(seed)
    N = n1 + 3 * n21 + 6 * n111
    for tries in range(1, max_tries + 1):
        p = [0.5 / N] if n1 else []
        for _ in range(n21):
            p += [0.5 / N * rng.uniform(0.3, 1.7), rng.uniform(0.02, 0.49)]
        for _ in range(n111):
            a = rng.uniform(0.02, 0.5)
            p += [0.5 / N * rng.uniform(0.3, 1.7), a, rng.uniform(0.02, (1 - a) / 2)]
        try:
            r = least_squares(res, np.array(p), method="lm", xtol=1e-15, ftol=1e-15, gtol=1e-15, max_nfev=3000)
        except Exception:
            continue
        if np.abs(r.fun).max() < 1e-11 and interior(r.x, n1, n21, n111):
            return r.x, tries
    raise SystemExit(f"no rule of degree {deg} found")


def interior(q, n1, n21, n111):
    k = 1 if n1 else 0
    ok = (q[0] > 0) if n1 else True
    for _ in range(n21):
        ok = ok and q[k] > 0 and 0 < q[k + 1] < 0.5
        k += 2
    for _ in range(n111):
        ok = ok and q[k] > 0 and q[k + 1] > 0 and q[k + 2] > 0 and q[k + 1] + q[k + 2] < 1
        k += 3
    return bool(ok)


def polish(p0, deg, n1, n21, n111):
    mp.mp.dps = 50
    IJ = invariants(deg)
    rhs = [mp.mpf(m.numerator) / mp.mpf(m.denominator) for m in exact_moments(deg)]

    def f(*p):
        t = orbit_terms(p, n1, n21, n111, one=mp.mpf(1))
        return [sum(w * e2 ** i * e3 ** j for w, e2, e3 in t) / rhs[n] - 1 for n, (i, j) in enumerate(IJ)]
    x = mp.findroot(f, [mp.mpf(float(v)) for v in p0], solver="mdnewton", tol=mp.mpf(10) ** -40, maxsteps=50)
    worst = max(abs(v) for v in f(*x))
    return [x[i] for i in range(len(p0))], worst


def canonical(p, n1, n21, n111):
    """orbits sorted by their parameter so the table does not depend on the start"""
    k = 1 if n1 else 0
    head = list(p[:k])
    s21 = sorted((tuple(p[k + 2 * i:k + 2 * i + 2]) for i in range(n21)), key=lambda t: t[1])
    k += 2 * n21
    s111 = []
    for i in range(n111):
        w, a, b = p[k + 3 * i:k + 3 * i + 3]
        abc = sorted([a, b, 1 - a - b])
        s111.append((w, abc[0], abc[1]))
    s111.sort(key=lambda t: (t[1], t[2]))
    return head + [v for t in s21 for v in t] + [v for t in s111 for v in t]


def main():
    out = sys.argv[1]
    specs = sys.argv[2:] or DEFAULT
    lines = ["// generated by tools/make_sym_rules.py: fully symmetric rules by moment fitting",
             "// {degree, n1, n21, n111, points, {w0?, (w, a) x n21, (w, a, b) x n111}}; weights sum to 1/2"]
    for s in specs:
        deg, n1, n21, n111 = (int(v) for v in s.split(":"))
        p0, tries = search(deg, n1, n21, n111)
        p, worst = polish(p0, deg, n1, n21, n111)
        p = canonical(p, n1, n21, n111)
        assert interior([float(v) for v in p], n1, n21, n111)
        npts = n1 + 3 * n21 + 6 * n111
        print(f"degree {deg}: {npts} points ({n1} + 3 x {n21} + 6 x {n111}), start {tries}, "
              f"worst relative moment residual {mp.nstr(worst, 3)}", flush=True)
        vals = ", ".join(mp.nstr(v, 20) for v in p)
        lines.append(f"{{{deg}, {n1}, {n21}, {n111}, {npts}, {{{vals}}}}},")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
