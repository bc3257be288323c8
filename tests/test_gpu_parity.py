"""GPU parity: libvp_b200.so (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star): near-field lists bit-exact; potentials within
1e-11 relative max-norm (||u_gpu - u_oracle||_inf / ||u_oracle||_inf, SURVEY.md
§9.9); deterministic counters (leaves, panels) identical.  Full-size configs
are checked on target samples (the oracle's far sum is O(T S))."""
import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from helpers import const_coeffs, small_mesh, tri_potential_const
from oracle.binding import Oracle

pytestmark = pytest.mark.gpu

REL_TOL = 1e-11


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def cfg1():
    pr = vp.load_config(1)
    ev = vp.Evaluator(0).load(pr)
    yield pr, ev, Oracle.from_problem(pr)
    ev.close()


@pytest.fixture(scope="module")
def cfg2():
    pr = vp.load_config(2)
    ev = vp.Evaluator(0).load(pr)
    yield pr, ev, Oracle.from_problem(pr)
    ev.close()


def assert_lists_equal(ev, O, txy):
    s_g, off_g, ids_g = ev.build_nearlist(txy)
    s_o, off_o, ids_o = O.nearlist(txy)
    assert np.array_equal(s_g, s_o), "S(t) differs"
    assert np.array_equal(off_g, off_o), "CSR offsets differ"
    assert np.array_equal(ids_g, ids_o), "N(t) ids differ"
    return s_o, off_o, ids_o


def test_lists_bit_exact_config1(cfg1):
    pr, ev, O = cfg1
    assert_lists_equal(ev, O, pr.txy)


def test_lists_bit_exact_config2(cfg2):
    pr, ev, O = cfg2
    assert_lists_equal(ev, O, pr.txy)


def test_sources_match(cfg2):
    pr, ev, O = cfg2
    sx, sy, q = ev.sources()
    osx, osy, oq = O.sources()
    assert np.abs(sx - osx).max() <= 2e-16 and np.abs(sy - osy).max() <= 2e-16
    assert rel(q, oq) <= 1e-14


def test_far_field_config1(cfg1):
    pr, ev, O = cfg1
    assert rel(ev.far_field(pr.txy), O.far_sum(pr.txy)) <= 1e-13


def test_far_field_config2_sample(cfg2):
    pr, ev, O = cfg2
    sub = pr.txy[::37]
    assert rel(ev.far_field(sub), O.far_sum(sub)) <= 1e-13


def test_u_config1_full(cfg1):
    pr, ev, O = cfg1
    u_g, st = ev.evaluate(pr.txy)
    u_o, _, sto = O.evaluate(pr.txy)
    assert rel(u_g, u_o) <= REL_TOL
    for k in ("n_near_pairs", "n_leaves", "n_panels", "n_self", "n_outside", "n_rho_le1", "n_degenerate",
              "max_depth"):
        assert st[k] == sto[k], k


def test_u_config2_sample(cfg2):
    pr, ev, O = cfg2
    u_g, st = ev.evaluate(pr.txy)
    sub = slice(3, None, 53)
    u_o, _, _ = O.evaluate(pr.txy[sub])
    assert rel(u_g[sub], u_o) <= REL_TOL


@pytest.mark.parametrize("far", ["direct", "fmm"])
def test_pair_stage_streams(cfg2, far):
    """Self pairs and point sums run on their own stream beside the near chain:
    the stage's wall time covers both and u does not depend on the far method
    beyond rounding (and is bit-identical run to run)."""
    pr, ev, _ = cfg2
    ev.set_far_method(far)
    try:
        u1, st = ev.evaluate(pr.txy)
        u2, _ = ev.evaluate(pr.txy)
    finally:
        ev.set_far_method("direct")
    assert np.array_equal(u1, u2)
    assert st["t_pair_ms"] > 0.0
    assert st["t_pair_ms"] >= max(st["t_near_ms"], st["t_self_ms"]) - 1e-3
    assert st["t_total_ms"] >= st["t_pair_ms"]


def test_near_pairs_per_pair(cfg2):
    pr, ev, O = cfg2
    s, off, ids = O.nearlist(pr.txy[::101])
    ts = np.repeat(np.arange(len(s)), np.diff(off))
    pick = np.linspace(0, len(ids) - 1, 200).astype(int)
    t = pr.txy[::101][ts[pick]]
    val, sub, lv = ev.near_pairs(t, ids[pick])
    ref = np.array([O.near_pair(x, y, e) for (x, y), e in zip(t, ids[pick])])
    scale = np.abs(ref[:, 1]).max()
    assert np.abs(val - ref[:, 0]).max() <= 1e-13 * scale
    assert np.abs(sub - ref[:, 1]).max() <= 1e-13 * scale
    assert np.array_equal(lv, ref[:, 2].astype(np.int64))


def test_self_pairs_per_pair(cfg2):
    pr, ev, O = cfg2
    tp = np.arange(0, pr.n_tgt, 911)
    s, _, _ = O.nearlist(pr.txy[tp])
    keep = s >= 0
    t, e = pr.txy[tp][keep], s[keep]
    val, sub, pn = ev.self_pairs(t, e)
    ref = np.array([O.self_pair(x, y, k) for (x, y), k in zip(t, e)])
    scale = np.abs(ref[:, 1]).max()
    assert np.abs(val - ref[:, 0]).max() <= 1e-13 * scale
    assert np.array_equal(pn, ref[:, 2].astype(np.int64))


def test_deterministic_and_shard_invariant(cfg2):
    """u is bit-identical run to run and per target whatever the shard."""
    pr, ev, _ = cfg2
    u1, _ = ev.evaluate(pr.txy)
    u2, _ = ev.evaluate(pr.txy)
    assert np.array_equal(u1, u2)
    for lo, hi in [(0, 50000), (50000, 120001), (120001, pr.n_tgt)]:
        us, _ = ev.evaluate(pr.txy[lo:hi])
        assert np.array_equal(us, u1[lo:hi])


def test_constant_density_closed_form_on_gpu(cfg1):
    pr, _, _ = cfg1
    with vp.Evaluator(0) as ev:
        ev.set_mesh(pr.vxy, pr.tri)
        ev.set_rules(pr.rules)
        ev.set_density(pr.p, const_coeffs(pr.n_tri, pr.p))
        u, _ = ev.evaluate(pr.txy)
    assert np.abs(u - tri_potential_const(pr.vxy, pr.tri, pr.txy)).max() <= 5e-12


def test_config3_sample_full_size():
    """Graded star mesh at full size (65,968 triangles), target sample."""
    pr = vp.load_config(3)
    O = Oracle.from_problem(pr)
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        sub = pr.txy[::4001]
        assert_lists_equal(ev, O, pr.txy[::97])
        u_g, _ = ev.evaluate(sub)
    u_o, _, _ = O.evaluate(sub)
    assert rel(u_g, u_o) <= REL_TOL


def test_edge_cases_small_mesh():
    vxy, tri = small_mesh()
    p = 3
    co = vp.project_density(vxy, tri, p, vp.F_LINEAR, [1.0, -0.5, 0.25])
    r = vp.make_rules(10)
    O = Oracle(vxy, tri, p, co, r)
    # outside, far outside, vertex, shared edge, boundary edge, interior
    txy = np.array([[2.0, 2.0], [-0.5, 0.5], [0.5, 0.5], [0.0, 0.0], [1.0, 0.0], [0.25, 0.0], [0.3, 0.3],
                    [0.7, 0.2], [1e-13, 0.4], [0.5, 1.0 + 1e-13]])
    with vp.Evaluator(0) as ev:
        ev.set_mesh(vxy, tri)
        ev.set_rules(r)
        ev.set_density(p, co)
        assert_lists_equal(ev, O, txy)
        u_g, st = ev.evaluate(txy)
        u_o, _, sto = O.evaluate(txy)
        assert rel(u_g, u_o) <= REL_TOL
        assert st["n_outside"] == sto["n_outside"] and st["n_leaves"] == sto["n_leaves"]
        assert st["n_panels"] == sto["n_panels"] and st["n_degenerate"] == sto["n_degenerate"]
        # empty target array
        u0, st0 = ev.evaluate(np.zeros((0, 2)))
        assert len(u0) == 0


@pytest.mark.parametrize("p", [0, 1, 2, 5, 12])
def test_density_orders(p):
    vxy, tri = small_mesh()
    co = np.random.default_rng(p).standard_normal((2, vp.koorn_size(p))) * 0.3
    r = vp.make_rules(8)
    O = Oracle(vxy, tri, p, co, r)
    lx, ly = vp.lattice_nodes(4)
    txy = np.concatenate([vxy[t[0]] + np.outer(lx, vxy[t[1]] - vxy[t[0]]) + np.outer(ly, vxy[t[2]] - vxy[t[0]])
                          for t in tri] + [np.array([[1.2, 0.5], [0.5, -0.05]])])
    with vp.Evaluator(0) as ev:
        ev.set_mesh(vxy, tri)
        ev.set_rules(r)
        ev.set_density(p, co)
        u_g, _ = ev.evaluate(txy)
    u_o, _, _ = O.evaluate(txy)
    assert rel(u_g, u_o) <= REL_TOL


def test_all_near_elements_list_parity():
    vxy, tri = small_mesh()
    co = const_coeffs(2, 1)
    r = vp.make_rules(6, eps=1.0)  # rho0 <= 1: all-near
    O = Oracle(vxy, tri, 1, co, r)
    txy = np.array([[5.0, 5.0], [0.2, 0.1], [0.9, 0.8], [-3.0, 0.5]])
    with vp.Evaluator(0) as ev:
        ev.set_mesh(vxy, tri)
        ev.set_rules(r)
        ev.set_density(1, co)
        assert_lists_equal(ev, O, txy)


def test_usage_errors():
    with vp.Evaluator(0) as ev:
        with pytest.raises(vp.UsageError):
            ev.evaluate(np.zeros((3, 2)))  # no mesh yet
        vxy, tri = small_mesh()
        with pytest.raises(vp.UsageError):
            ev.set_mesh(vxy, tri[:, ::-1])  # clockwise
        with pytest.raises(vp.UsageError):
            ev.set_mesh(vxy, np.array([[0, 1, 7]]))
        ev.set_mesh(vxy, tri)
        with pytest.raises(vp.UsageError):
            ev.set_density(13, np.zeros((2, 105)))


def test_config4_full_size_target_sample():
    """1,048,576-triangle jittered square with staggered targets (some
    outside, S = -1): lists on a sample, u on a small sample."""
    pr = vp.load_config(4)
    O = Oracle.from_problem(pr)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(pr.n_tgt, 2000, replace=False))
    edge = np.nonzero(pr.txy[:, 0] > 1.0)[0][:50]  # outside the square
    sample = pr.txy[np.concatenate([idx, edge])]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        s, _, _ = assert_lists_equal(ev, O, sample)
        assert (s == -1).any()
        u_g, _ = ev.evaluate(sample[::40])
    u_o, _, _ = O.evaluate(sample[::40])
    assert rel(u_g, u_o) <= REL_TOL


# ---------------------------------------------------------------------------
# FMM far field: same parity bar as the direct path

@pytest.mark.parametrize("cfg,stride", [(1, 1), (2, 53)])
def test_fmm_evaluation_matches_oracle(cfg, stride):
    pr = vp.load_config(cfg)
    O = Oracle.from_problem(pr)
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ev.set_far_method("fmm")
        u_g, st = ev.evaluate(pr.txy)
        assert st["far_method"] == 1 and st["fmm_levels"] >= 2
    sub = slice(1, None, stride)
    u_o, _, _ = O.evaluate(pr.txy[sub])
    assert rel(u_g[sub], u_o) <= REL_TOL


def test_fmm_far_field_outside_targets_and_determinism(cfg2):
    pr, ev, O = cfg2
    t = np.vstack([pr.txy[::211], [[5.0, 5.0], [-3.0, 0.25], [0.0, 1.5]]])
    ev.set_far_method("fmm", 40)
    try:
        uf = ev.far_field(t)
        uf2 = ev.far_field(t)
        u1, st = ev.evaluate(t)
        u_half, _ = ev.evaluate(t[: len(t) // 2])
    finally:
        ev.set_far_method("direct")
    assert np.array_equal(uf, uf2)
    assert np.array_equal(u_half, u1[: len(t) // 2])  # shard invariance (tree from sources only)
    assert rel(uf, O.far_sum(t)) <= 1e-12
    assert st["fmm_outside"] >= 2


def test_coincident_target_and_source():
    """A target placed exactly on a far-rule node of its own element: the
    coincident pair contributes 0 in every path."""
    pr = vp.load_config(1)
    O = Oracle.from_problem(pr)
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        sx, sy, _ = ev.sources()
        t = np.stack([sx[[0, 100, 5000]], sy[[0, 100, 5000]]], 1)
        t = np.vstack([t, pr.txy[:50]])
        u_d, _ = ev.evaluate(t)
        uf_d = ev.far_field(t)
        ev.set_far_method("fmm")
        u_f, _ = ev.evaluate(t)
    u_o, uf_o, _ = O.evaluate(t)
    assert rel(uf_d, uf_o) <= 1e-13
    assert rel(u_d, u_o) <= REL_TOL and rel(u_f, u_o) <= REL_TOL


@pytest.mark.parametrize("depth", [-1, 0, 1, 3])
def test_near_cache_depths_match_oracle(cfg2, depth):
    """The per-element near-leaf density cache (any depth, or off) leaves the
    near corrections at oracle parity and the leaf counts unchanged."""
    pr, ev, O = cfg2
    s, off, ids = O.nearlist(pr.txy[::151])
    ts = np.repeat(np.arange(len(s)), np.diff(off))
    pick = np.linspace(0, len(ids) - 1, 120).astype(int)
    t = pr.txy[::151][ts[pick]]
    ev.set_near_cache(depth)
    try:
        val, sub, lv = ev.near_pairs(t, ids[pick])
        u, _ = ev.evaluate(pr.txy[::97])
    finally:
        ev.set_near_cache(3)
    ref = np.array([O.near_pair(x, y, e) for (x, y), e in zip(t, ids[pick])])
    scale = np.abs(ref[:, 1]).max()
    assert np.abs(val - ref[:, 0]).max() <= 1e-13 * scale
    assert np.array_equal(lv, ref[:, 2].astype(np.int64))
    u_o, _, _ = O.evaluate(pr.txy[::97])
    assert rel(u, u_o) <= REL_TOL


# ---------------------------------------------------------------------------
# Potential interpolation: interp_coeffs + field_eval

def test_interp_reproduces_polynomials_and_matches_numpy():
    from oracle import binding as ob
    vxy, tri = small_mesh()
    p = 4
    lx, ly = vp.lattice_nodes(p)
    M = vp.koorn_size(p)
    poly = lambda x, y: 0.3 + x - 2 * y + x * y ** 2 - 0.5 * x ** 4 + y ** 3 * x  # noqa: E731  degree 4
    P = vxy[tri]
    nodes = P[:, 0, None, :] + lx[None, :, None] * (P[:, 1] - P[:, 0])[:, None, :] + \
        ly[None, :, None] * (P[:, 2] - P[:, 0])[:, None, :]
    vals = poly(nodes[..., 0], nodes[..., 1])
    with vp.Evaluator(0) as ev:
        co, cond = ev.interp_coeffs(p, lx, ly, vals)
        V = np.array([ob.koornwinder(p, x, y) for x, y in zip(lx, ly)])
        ref = np.linalg.solve(V, vals.T).T
        assert np.abs(co - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
        assert 1.0 <= cond < 1e6
        rng = np.random.default_rng(3)
        pts = rng.random((500, 2))
        f, eo = ev.field_eval(vxy, tri, p, co, pts)
        assert (eo >= 0).all()
        assert np.abs(f - poly(pts[:, 0], pts[:, 1])).max() <= cond * 1e-13
        f2, eo2 = ev.field_eval(vxy, tri, p, co, np.array([[2.0, 2.0], [0.5, 0.25]]), allow_outside=True)
        assert eo2[0] == -1 and np.isnan(f2[0]) and eo2[1] == 0
        with pytest.raises(vp.NumericalError):
            ev.field_eval(vxy, tri, p, co, np.array([[2.0, 2.0]]))


def test_potential_field_of_config1(cfg1):
    """evaluate_field phase 3: u at the interpolation nodes -> PotentialField ->
    field_eval reproduces the nodal values and approximates u elsewhere."""
    pr, ev, O = cfg1
    u, _ = ev.evaluate(pr.txy)
    lx, ly = vp.lattice_nodes(pr.p)
    co, cond = ev.interp_coeffs(pr.p, lx, ly, u.reshape(pr.n_tri, -1))
    f, eo = ev.field_eval(pr.vxy, pr.tri, pr.p, co, pr.txy)
    assert np.abs(f - u).max() <= cond * 1e-13 * np.abs(u).max()
    rng = np.random.default_rng(5)
    pts = 0.05 + 0.9 * rng.random((64, 2))
    fi, _ = ev.field_eval(pr.vxy, pr.tri, pr.p, co, pts)
    u_o, _, _ = O.evaluate(pts)
    assert np.abs(fi - u_o).max() <= 1e-5 * np.abs(u_o).max()


# ---------------------------------------------------------------------------
# Ball near-field baseline

@pytest.mark.parametrize("cfg,stride", [(1, 3), (2, 61)])
def test_ball_model_lists_and_u_match_oracle(cfg, stride):
    pr = vp.load_config(cfg)
    O = Oracle.from_problem(pr, near_model=1, ball_factor=1.5)
    sub = pr.txy[::stride]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ev.set_near_model("ball", 1.5)
        assert_lists_equal(ev, O, pr.txy)
        u_g, st = ev.evaluate(sub)
    u_o, _, sto = O.evaluate(sub)
    assert rel(u_g, u_o) <= REL_TOL
    assert st["n_leaves"] == sto["n_leaves"] and st["n_near_pairs"] == sto["n_near_pairs"]


@pytest.mark.parametrize("q", [10, 24])
def test_config5_q_sweep_sample(q):
    """Config 5 (262k-triangle graded star) at the sweep's extreme far orders."""
    pr = vp.load_config(5, q)
    O = Oracle.from_problem(pr)
    sub = pr.txy[::200003]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        assert_lists_equal(ev, O, pr.txy[::40009])
        u_g, st = ev.evaluate(sub)
    u_o, _, sto = O.evaluate(sub)
    assert rel(u_g, u_o) <= REL_TOL
    assert st["n_leaves"] == sto["n_leaves"] and st["n_panels"] == sto["n_panels"]


def test_p12_on_config1_mesh():
    pr = vp.load_config(1)
    co = vp.project_density(pr.vxy, pr.tri, 12, vp.F_SQUARE)
    r = vp.make_rules(14)
    O = Oracle(pr.vxy, pr.tri, 12, co, r)
    sub = pr.txy[::11]
    with vp.Evaluator(0) as ev:
        ev.set_mesh(pr.vxy, pr.tri)
        ev.set_rules(r)
        ev.set_density(12, co)
        u_g, _ = ev.evaluate(sub)
    u_o, _, _ = O.evaluate(sub)
    assert rel(u_g, u_o) <= REL_TOL


_VARIANT_SCRIPT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2205_04401_b200 as vp
pr = vp.load_config(2)
with vp.Evaluator(0) as ev:
    ev.load(pr)
    u, st = ev.evaluate(pr.txy[::7])
np.save({out!r}, u)
"""


@pytest.mark.parametrize("env", [{"VP_NEAR_CT": "1"}, {"VP_NEAR_CG": "1"}, {"VP_NEAR_CACHE_SIMT": "1"}])
def test_near_kernel_variants_agree(tmp_path, env):
    """The one-leaf and leaf-group cached-leaf kernels (k_near_ct, k_near_cg)
    and the DFMA near-cache contraction (k_near_cache) -- the A/B
    alternatives of k_near_c8 and the DMMA k_near_cache_mma -- give the same
    u up to summation order."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for k, e in enumerate([{}, env]):
        out = str(tmp_path / f"u{k}.npy")
        subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT.format(root=root, out=out)], check=True,
                       env={**os.environ, **e}, timeout=600)
        outs.append(np.load(out))
    assert rel(outs[1], outs[0]) <= 1e-13


def test_nonfinite_target_is_a_numerical_error(cfg1):
    """A NaN or infinite target coordinate fails the evaluation with code 2
    (numerical failure; the check runs on the device in the list build), and
    the context keeps working afterwards."""
    pr, ev, O = cfg1
    for bad in (np.nan, np.inf):
        txy = pr.txy[:64].copy()
        txy[17, 1] = bad
        with pytest.raises(vp.NumericalError, match="non-finite"):
            ev.evaluate(txy)
    u, _ = ev.evaluate(pr.txy[:64])
    u_o, _, _ = O.evaluate(pr.txy[:64])
    assert rel(u, u_o) <= REL_TOL
