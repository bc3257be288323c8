"""GPU parity, round 2: wider full-size samples, the user-stream device
entry point, the corrections-only far method, the near-depth guarantee and
the multi-GPU plan / gather entry points (through the C-ABI).

Bar as in test_gpu_parity.py: lists bit-exact, u within 1e-11 relative
max-norm of the CPU oracle, deterministic counters equal."""
import ctypes

import numpy as np
import pytest

import paper_2205_04401_b200 as vp
from paper_2205_04401_b200.dist import morton_order
from oracle.binding import Oracle

pytestmark = pytest.mark.gpu

REL_TOL = 1e-11


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def boundary_and_spread(pr, n_edge, n_spread, seed=0):
    """n_edge targets nearest the domain boundary (graded, finest elements;
    outside targets for staggered meshes) + n_spread uniform ones."""
    rng = np.random.default_rng(seed)
    if pr.config == 4:
        d = np.minimum.reduce([pr.txy[:, 0], 1 - pr.txy[:, 0], pr.txy[:, 1], 1 - pr.txy[:, 1]])
    else:  # star / disk: boundary radius along the ray
        th = np.arctan2(pr.txy[:, 1], pr.txy[:, 0])
        rb = 1.0 + 0.3 * np.cos(5 * th) if pr.config in (3, 5) else np.ones(len(th))
        d = rb - np.hypot(pr.txy[:, 0], pr.txy[:, 1])
    edge = np.argsort(d, kind="stable")[:n_edge]
    spread = rng.choice(pr.n_tgt, n_spread, replace=False)
    return np.unique(np.concatenate([edge, spread]))


@pytest.mark.parametrize("cfg,q", [(3, 0), (4, 0), (5, 16)])
def test_full_size_u_500_targets(cfg, q):
    """>= 500 targets per full-size config: 250 nearest the boundary (the
    graded band of configs 3/5; outside-the-square targets of config 4) and
    250 uniform.  Config 5 at its default q = 16."""
    pr = vp.load_config(cfg, q)
    O = Oracle.from_problem(pr)
    idx = boundary_and_spread(pr, 250, 260, seed=cfg)
    assert len(idx) >= 500
    t = pr.txy[idx]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        s_g, off_g, ids_g = ev.build_nearlist(t)
        u_g, st = ev.evaluate(t)
    s_o, off_o, ids_o = O.nearlist(t)
    assert np.array_equal(s_g, s_o) and np.array_equal(off_g, off_o) and np.array_equal(ids_g, ids_o)
    u_o, _, sto = O.evaluate(t)
    assert rel(u_g, u_o) <= REL_TOL
    for k in ("n_leaves", "n_panels", "n_near_pairs", "n_self", "n_rho_le1", "n_degenerate"):
        assert st[k] == sto[k], k


def test_evaluate_device_on_user_stream():
    """vp_evaluate_device (the entry bench.py times) on a caller's stream:
    bitwise equal to vp_evaluate, within 1e-11 of the oracle."""
    import torch
    pr = vp.load_config(2)
    t = pr.txy[::7]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        u_h, _ = ev.evaluate(t)
        s = torch.cuda.Stream()
        d_t = torch.from_numpy(t).cuda()
        d_u = torch.full((len(t),), np.nan, dtype=torch.float64, device="cuda")
        with torch.cuda.stream(s):
            busy = torch.empty(1 << 26, device="cuda").normal_()  # queued work ahead on the user stream
            st = ev.evaluate_device(len(t), d_t.data_ptr(), d_u.data_ptr(), s.cuda_stream)
        s.synchronize()
        u_d = d_u.cpu().numpy()
        del busy
    assert st["n_targets"] == len(t)
    assert np.array_equal(u_d, u_h)
    u_o, _, _ = Oracle.from_problem(pr).evaluate(t[::5])
    assert rel(u_d[::5], u_o) <= REL_TOL


def test_far_method_none_gives_the_corrections():
    """Far method 'none' returns sum (I_T - point sum) over N(t) and S(t): adding
    the direct far field recovers the full u."""
    pr = vp.load_config(2)
    t = pr.txy[::11]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        u_full, _ = ev.evaluate(t)
        ev.set_far_method("none")
        u_corr, st = ev.evaluate(t)
        ev.set_far_method("direct")
        u_far = ev.far_field(t)
    assert st["far_method"] == 2
    assert np.abs(u_corr + u_far - u_full).max() <= 1e-14 * np.abs(u_full).max()


def test_near_depth_bound_refused_and_near_edge_target():
    """leaf path codes hold 29 levels.  An element whose N_n model
    could need a deeper near_eval is refused at vp_set_rules (status 2); a
    target 1e-10 h outside a neighbour's edge evaluates and matches the
    oracle (its recursion stops where rho_d <= 1)."""
    from helpers import small_mesh
    vxy, tri = small_mesh()
    p = 3
    co = vp.project_density(vxy, tri, p, vp.F_SQUARE)
    # huge elements at tiny eps: rho0(N_n) = (w_edge |J| / (eps C_12))^(1/12) > 28.5
    ev = vp.Evaluator(0)
    ev.set_mesh(vxy * 1e6, tri)
    with pytest.raises(vp.NumericalError):
        ev.set_rules(vp.make_rules(8, eps=1e-16))
    with pytest.raises(vp.UsageError):
        ev.set_density(p, co)
        ev.evaluate(np.zeros((1, 2)))
    ev.close()
    r = vp.make_rules(8, eps=1e-12)
    a, b = vxy[tri[0, 0]], vxy[tri[0, 1]]
    m = 0.5 * (a + b)
    nrm = np.array([b[1] - a[1], a[0] - b[0]])
    nrm /= np.hypot(*nrm)
    h = np.hypot(*(b - a))
    t = np.stack([m + 1e-10 * h * nrm, m - 1e-10 * h * nrm, a + 3e-11 * h * nrm])
    with vp.Evaluator(0) as ev:
        ev.set_mesh(vxy, tri)
        ev.set_rules(r)
        ev.set_density(p, co)
        u_g, st = ev.evaluate(t)
    O = Oracle(vxy, tri, p, co, r)
    u_o, _, sto = O.evaluate(t)
    assert rel(u_g, u_o) <= REL_TOL
    assert st["n_leaves"] == sto["n_leaves"] and st["max_depth"] == sto["max_depth"]
    assert st["max_depth"] <= 29


def test_shard_plan_morton_balance_and_bitwise_gather():
    """vp_shard_plan: the Morton order is dist.morton_order's; the bounds
    split the cost evenly; evaluating the shards separately and gathering
    them reproduces the one-shot u bit for bit."""
    pr = vp.load_config(2)
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        u_all, _ = ev.evaluate(pr.txy)
        for world in (1, 3, 8):
            order, bounds, cost = ev.shard_plan(pr.txy, world)
            assert np.array_equal(order.astype(np.int64), morton_order(pr.txy))
            assert bounds[0] == 0 and bounds[-1] == pr.n_tgt and np.all(np.diff(bounds) >= 0)
            assert cost.sum() > 0 and cost.max() <= cost.sum() / world * 1.01 + 1e6
            parts = [ev.evaluate(pr.txy[order[bounds[r]:bounds[r + 1]]])[0] for r in range(world)]
            assert np.array_equal(np.concatenate(parts), u_all[order])
        # FMM costs differ from direct ones, but the plan still partitions
        ev.set_far_method("fmm")
        _, b2, c2 = ev.shard_plan(pr.txy, 4)
        assert b2[-1] == pr.n_tgt and c2.max() <= c2.sum() / 4 * 1.05


def test_comm_world1_gather_and_stats():
    """The library's NCCL communicator at world size 1: vp_gather places the
    shard, vp_allreduce_stats is the identity."""
    import torch
    pr = vp.load_config(1)
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ev.comm_init(1, 0, vp.nccl_unique_id())
        d_t = torch.from_numpy(pr.txy).cuda()
        d_u = torch.empty(pr.n_tgt, dtype=torch.float64, device="cuda")
        d_all = torch.zeros(pr.n_tgt, dtype=torch.float64, device="cuda")
        st = ev.evaluate_device(pr.n_tgt, d_t.data_ptr(), d_u.data_ptr(), 0)
        ev.gather(np.array([0, pr.n_tgt]), d_u.data_ptr(), d_all.data_ptr(), 0)
        torch.cuda.synchronize()
        assert torch.equal(d_all, d_u)
        st2 = ev.allreduce_stats(st)
        for k in ("n_targets", "n_near_pairs", "n_leaves", "n_panels"):
            assert st2[k] == st[k]
        assert abs(st2["t_total_ms"] - st["t_total_ms"]) < 1e-9


@pytest.mark.parametrize("far", ["direct", "fmm", "none"])
def test_graph_replay_matches_eager(far):
    """vp_evaluate_graph: the captured evaluation (no host round trips)
    reproduces the eager one bit for bit, also after vp_set_density with new
    coefficients of the same order, and vp_graph_status reports its counters."""
    import torch
    pr = vp.load_config(2)
    t = np.ascontiguousarray(pr.txy[::5])
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ev.set_far_method(far)
        u_e, st_e = ev.evaluate(t)
        d_t = torch.from_numpy(t).cuda()
        d_u = torch.zeros(len(t), dtype=torch.float64, device="cuda")
        s = torch.cuda.Stream()
        for _ in range(3):
            ev.evaluate_graph(len(t), d_t.data_ptr(), d_u.data_ptr(), s.cuda_stream)
        st_g = ev.graph_status(s.cuda_stream)
        assert np.array_equal(d_u.cpu().numpy(), u_e)
        for k in ("n_near_pairs", "n_leaves", "n_panels", "n_self", "n_rho_le1", "max_depth"):
            assert st_g[k] == st_e[k], k
        c2 = pr.coeffs * 0.5 + 0.25 * np.roll(pr.coeffs, 7, axis=0)
        ev.set_density(pr.p, c2)
        u_e2, _ = ev.evaluate(t)
        ev.evaluate_graph(len(t), d_t.data_ptr(), d_u.data_ptr(), s.cuda_stream)
        ev.graph_status(s.cuda_stream)
        assert np.array_equal(d_u.cpu().numpy(), u_e2)


def test_cpp_caller_on_gpu(tmp_path):
    """The C++ caller (no Python in the process): config 1 through vp.h, the
    two vp_shard_plan shards bitwise equal to the one-shot u, u within 1e-11
    of the oracle."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["make", "-C", root, "abi-caller"], check=True, capture_output=True)
    out = str(tmp_path / "u.bin")
    r = subprocess.run([os.path.join(root, "tests", "cpp", "vp_abi_caller"), out, "1"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "bitwise equal" in r.stdout
    u = np.fromfile(out, dtype=np.float64)
    pr = vp.load_config(1)
    assert u.size == pr.n_tgt
    u_o, _, _ = Oracle.from_problem(pr).evaluate(pr.txy[::3])
    assert rel(u[::3], u_o) <= REL_TOL
