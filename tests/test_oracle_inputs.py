"""The oracle's own inputs (oracle/vp_oracle_inputs.cpp) against the product's
host generators (vp_setup.cpp, in libvp_b200.so).

The oracle builds every configuration, rule and density projection itself,
so the reference arm of bench.py and the oracle side of the parity tests do
not depend on the product library.  These tests pin the two generators to
each other: meshes, targets and density parameters byte for byte, rules to
rounding (GGQ bit for bit), coefficients to rounding.  No GPU needed.
"""
import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from oracle import binding as B


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_bytes_equal(cfg):
    P = B.OracleProblem(cfg)
    Q = vp.load_config(cfg, with_rules=False)
    assert (P.p, P.q, P.eps, P.density_kind, P.staggered) == (Q.p, Q.q, Q.eps, Q.density_kind, Q.staggered)
    assert P.vxy.tobytes() == Q.vxy.tobytes()
    assert P.tri.tobytes() == Q.tri.tobytes()
    assert P.txy.tobytes() == Q.txy.tobytes()
    assert P.params.tobytes() == Q.params.tobytes()
    # coefficients: same projection with rules equal to one ulp
    scale = np.abs(Q.coeffs).max()
    assert np.abs(P.coeffs - Q.coeffs).max() <= 4e-15 * scale


def test_config_q_override_and_errors():
    P = B.OracleProblem(5, q_override=24)
    assert P.q == 24 and P.rules.q == 24
    with pytest.raises(B.OracleError) as e:
        B.OracleProblem(6)
    assert e.value.code == 1


@pytest.mark.parametrize("q", [6, 10, 12, 16, 20, 24, 40])
def test_simplex_rule_matches_product(q):
    a = B.simplex_rule(q)
    b = vp.simplex_rule(q)
    for x, y in zip(a, b):  # nodes to one ulp of 1, weights to a few ulps
        assert np.abs(x - y).max() <= 2.3e-16
    B.validate_rule(min(q, 32), *a)  # the reference's validate_rule contract (rules.hpp:60-85)


@pytest.mark.parametrize("q", [6, 10, 12, 16, 24])
def test_quad_rule_matches_product(q):
    """The evaluation's rule: the oracle expands its own copy of the orbit
    table (symmetric rules bit for bit); other orders as simplex_rule."""
    a, b = B.quad_rule(q), vp.quad_rule(q)
    assert len(a[0]) == len(b[0])
    if q in (6, 10, 12):
        assert all(u.tobytes() == v.tobytes() for u, v in zip(a, b))
    else:
        assert all(np.abs(u - v).max() <= 2.3e-16 for u, v in zip(a, b))
    B.validate_rule(q, *a)


@pytest.mark.parametrize("ng", [2, 5, 8])
def test_ggq_matches_product(ng):
    r, w, res = B.ggq(ng)
    r2, w2, res2 = vp.build_ggq(ng)
    assert r.tobytes() == r2.tobytes() and w.tobytes() == w2.tobytes()
    assert res <= 1e-13
    # the reference's analytic moments (test_basis.cpp:182-183)
    assert abs(np.sum(w * r) - 0.5) < 1e-14
    assert abs(np.sum(w * r * np.log(r)) + 0.25) < 1e-14


def test_gauss_jacobi_moments():
    # int_0^1 (1-u) u^k du = 1/((k+1)(k+2)), exact for k <= 2n-1
    for n in (1, 3, 7, 13):
        x, w = B.gauss_jacobi10(n)
        for k in range(2 * n):
            assert abs(np.sum(w * x ** k) - 1.0 / ((k + 1) * (k + 2))) < 1e-15


def test_lattice_and_density_eval_match():
    for p in (0, 4, 8, 12):
        a = B.lattice_nodes(p)
        b = vp.lattice_nodes(p)
        assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    P = B.OracleProblem(3)
    for x, y in [(0.1, 0.2), (-0.5, 0.7), (1.1, 0.0)]:
        assert B.lib().vpo_density_eval(3, B._d(P.params), P.params.size, x, y) == \
            vp.density_eval(3, P.params, x, y)


def test_oracle_on_own_inputs_equals_product_inputs():
    """The oracle evaluated on its own inputs and on the product's agrees to
    rounding (config 1, every target): the inputs are interchangeable."""
    P = B.OracleProblem(1)
    Q = vp.load_config(1)
    uo, _, so = B.Oracle.from_problem(P).evaluate(P.txy)
    up, _, sp = B.Oracle.from_problem(Q).evaluate(Q.txy)
    assert np.abs(uo - up).max() <= 1e-13 * np.abs(up).max()
    for k in ("n_near_pairs", "n_self", "n_leaves", "n_panels"):
        assert so[k] == sp[k]


def test_persistent_context_equals_one_shot():
    P = B.OracleProblem(2)
    O = B.Oracle.from_problem(P)
    sub = P.txy[::997]
    u1, uf1, s1 = O.evaluate(sub)
    ctx = O.open()
    for _ in range(2):
        u2, uf2, s2 = ctx.evaluate(sub)
        assert u1.tobytes() == u2.tobytes() and uf1.tobytes() == uf2.tobytes()
        assert s1 == s2
    ctx.close()
