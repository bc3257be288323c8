"""Quick GPU-vs-oracle comparison (development aid; tests/ hold the gates)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2205_04401_b200 as vp
from oracle.binding import Oracle

def check(cfg, stride):
    pr = vp.load_config(cfg)
    O = Oracle.from_problem(pr)
    ev = vp.Evaluator(0).load(pr)
    sub = pr.txy[::stride]
    s_g, off_g, ids_g = ev.build_nearlist(pr.txy)
    s_o, off_o, ids_o = O.nearlist(pr.txy)
    print(f"cfg{cfg} lists: self eq {np.array_equal(s_g, s_o)} off eq {np.array_equal(off_g, off_o)} "
          f"ids eq {np.array_equal(ids_g, ids_o)} n_ids {len(ids_g)} vs {len(ids_o)}", flush=True)
    sx, sy, q = ev.sources(); osx, osy, oq = O.sources()
    print(f"  sources max rel err q {np.abs(q - oq).max() / np.abs(oq).max():.3e} xy {np.abs(sx - osx).max():.3e}")
    uf_g = ev.far_field(sub); uf_o = O.far_sum(sub)
    print(f"  far rel err {np.abs(uf_g - uf_o).max() / np.abs(uf_o).max():.3e}", flush=True)
    t = time.time(); u_g, st = ev.evaluate(pr.txy); tg = time.time() - t
    t = time.time(); u_o, uf, sto = O.evaluate(sub); to = time.time() - t
    err = np.abs(u_g[::stride] - u_o).max() / np.abs(u_o).max()
    print(f"  u rel err {err:.3e}  gpu {tg*1e3:.1f} ms (dev {st['t_total_ms']:.2f} ms: list {st['t_list_ms']:.2f} far {st['t_far_ms']:.2f} near {st['t_near_ms']:.2f} self {st['t_self_ms']:.2f})  oracle {to:.2f}s on {len(sub)}")
    print("  gpu stats", {k: st[k] for k in ('n_near_pairs', 'n_leaves', 'n_panels', 'n_self', 'n_rho_le1', 'n_degenerate', 'max_depth')})
    print("  ora stats", sto)
    # per-pair near/self at a few pairs
    ts = np.repeat(np.arange(len(s_o)), np.diff(off_o))
    pick = np.linspace(0, len(ids_o) - 1, min(64, len(ids_o))).astype(int)
    v, sb, lv = ev.near_pairs(pr.txy[ts[pick]], ids_o[pick])
    ov = np.array([O.near_pair(*pr.txy[ts[i]], ids_o[i]) for i in pick])
    print(f"  near pair max abs err {np.abs(v - ov[:, 0]).max():.3e} sub {np.abs(sb - ov[:, 1]).max():.3e} leaves eq {np.array_equal(lv, ov[:, 2].astype(int))}")
    tp = np.linspace(0, len(s_o) - 1, 64).astype(int)
    tp = tp[s_o[tp] >= 0]
    v, sb, pn = ev.self_pairs(pr.txy[tp], s_o[tp])
    ov = np.array([O.self_pair(*pr.txy[i], s_o[i]) for i in tp])
    print(f"  self pair max abs err {np.abs(v - ov[:, 0]).max():.3e} sub {np.abs(sb - ov[:, 1]).max():.3e} panels eq {np.array_equal(pn, ov[:, 2].astype(int))}", flush=True)

check(1, 1)
check(2, 61)
