"""GPU parity, round 3 work: the self kernel's monomial density samples.

K5 (k_self) samples the density of an element from its monomial
coefficients about the reference centroid for p <= 8 (k_mono).  For smooth
densities this is as accurate as the Koornwinder recurrence; for rough ones
(unit-normal Koornwinder coefficients) the monomial basis amplifies rounding
by its coefficient growth, ~1e2 at p = 6 and ~1e3 at p = 8, which this test
bounds per pair at 1e-12 of the pair scale (the evaluation bar stays 1e-11
relative on u, test_density_orders)."""
import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from oracle.binding import Oracle
from helpers import small_mesh

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p", [4, 6, 8])
def test_self_pairs_rough_density(p):
    vxy, tri = small_mesh()
    co = np.random.default_rng(10 + p).standard_normal((2, vp.koorn_size(p)))
    r = vp.make_rules(2 * p)
    O = Oracle(vxy, tri, p, co, r)
    rng = np.random.default_rng(p)
    pts, elem = [], []
    for e, t in enumerate(tri):
        a, b = rng.random((2, 40))
        m = a + b < 1.0
        a, b = a[m], b[m]
        pts.append(vxy[t[0]] + np.outer(a, vxy[t[1]] - vxy[t[0]]) + np.outer(b, vxy[t[2]] - vxy[t[0]]))
        elem.append(np.full(len(a), e, dtype=np.int32))
    t, e = np.concatenate(pts), np.concatenate(elem)
    with vp.Evaluator(0) as ev:
        ev.set_mesh(vxy, tri)
        ev.set_rules(r)
        ev.set_density(p, co)
        val, sub, pn = ev.self_pairs(t, e)
    ref = np.array([O.self_pair(x, y, k) for (x, y), k in zip(t, e)])
    scale = np.abs(ref[:, 0]).max()
    assert np.abs(val - ref[:, 0]).max() <= 1e-12 * scale
    assert np.array_equal(pn, ref[:, 2].astype(np.int64))
