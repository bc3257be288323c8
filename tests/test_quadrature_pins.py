"""Independent pins of the hot path's quadrature: the oracle's near_eval and
self_eval (the algorithm the GPU reproduces to 1e-13 per pair,
tests/test_gpu_parity.py) against an adaptive long-double integration of the
same integral (oracle/vp_oracle_accept.cpp: recursive 4-way subdivision with
a 256-node order-30 rule), on random triangles with random order-6
densities.  SURVEY.md §4 test plan item 4 ("independent adaptive quadrature
of selected (target, triangle) pairs"), for polynomial densities of the
configs' order instead of the linear f of tests/test_oracle_kat.py.

- near_eval at targets 0.3 h down to 1e-8 h outside an
  edge: every accepted leaf is within eps (1e-12) of its integral by the
  near-field model, and a pair sums up to ~90 leaves; measured worst 6.8 eps
  in int log|x-y| f dA over 6 triangles x 24 targets (bar 10 eps).
- self_eval at targets inside, near an edge (1e-6 h,
  1e-10 h), near a vertex and at the centroid: agreement to 1e-14 relative
  (GGQ x Gauss-Legendre vs adaptive; measured 5e-15).
No GPU needed."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import soundness_sweep as S  # noqa: E402
from oracle import binding as B  # noqa: E402

P, EPS = 6, 1e-12


def cases(n=6, seed=11):
    rng = np.random.default_rng(seed)
    out = [np.array([0.0, 0.0, 0.05, 0.0, 0.0, 0.05])]
    for t in S.random_triangles(n - 1, seed=seed):
        out.append(t * 0.05)  # element scale of the BASELINE meshes
    M = (P + 1) * (P + 2) // 2
    return [(t, np.array([rng.uniform(-1, 1) * 0.5 ** n for n in range(P + 1) for m in range(n + 1)]))
            for t in out]


def oracle_of(tri, c):
    return B.Oracle(tri.reshape(3, 2), np.array([[0, 1, 2]], dtype=np.int32), P, c, B.OracleRules(12, eps=EPS))


@pytest.mark.parametrize("k", range(6))
def test_near_eval_within_eps_of_adaptive(k):
    tri, c = cases()[k]
    O = oracle_of(tri, c)
    v = tri.reshape(3, 2)
    for side in range(3):
        a, b = v[side], v[(side + 1) % 3]
        h = np.hypot(*(b - a))
        e = (b - a) / h
        nrm = np.array([e[1], -e[0]])
        if np.dot(v.mean(0) - 0.5 * (a + b), nrm) > 0:
            nrm = -nrm
        for d in (0.3, 1e-2, 1e-5, 1e-8):
            for s in (0.5, 0.17):
                t = a + s * (b - a) + d * h * nrm
                val, _, leaves, _ = O.near_pair(t[0], t[1], 0)
                ex = B.adaptive_log_integral(tri, 3, t[None], coeffs=c, p=P)[0] / (2 * np.pi)
                assert abs(val - ex) * 2 * np.pi <= 10 * EPS, (side, d, s, val, ex, leaves)


@pytest.mark.parametrize("k", range(6))
def test_self_eval_matches_adaptive(k):
    tri, c = cases()[k]
    O = oracle_of(tri, c)
    v = tri.reshape(3, 2)
    cen = v.mean(0)
    pts = [cen, 0.98 * v[0] + 0.02 * cen, 0.999 * v[2] + 0.001 * cen]
    for side in range(3):
        a, b = v[side], v[(side + 1) % 3]
        inward = cen - 0.5 * (a + b)
        for d in (1e-6, 1e-10):
            pts.append(a + 0.37 * (b - a) + d * inward / np.hypot(*inward) * np.hypot(*(b - a)))
    for t in pts:
        val, _, panels = O.self_pair(t[0], t[1], 0)
        ex = B.adaptive_log_integral(tri, 3, np.asarray(t)[None], coeffs=c, p=P)[0] / (2 * np.pi)
        assert abs(val - ex) <= 1e-13 * abs(ex), (t, val, ex, panels)
