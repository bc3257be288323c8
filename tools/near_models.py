"""Precise (Bernstein-ellipse) vs ball near-field model on the unit disk
(config 2 mesh and staggered targets, f = 1 so the exact potential of the
polygonal disk is known in closed form): corrections per target c, near
leaves per target s_n, arc-length panels s_l and the max error, for the
paper's tolerance sweep (PAPER.md Table near_corr; SPEC acceptance 1-2).

  python tools/near_models.py [--out profiles/r01_near_models.json]
"""
import argparse, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2205_04401_b200 as vp  # noqa: E402
from helpers import const_coeffs, tri_potential_const  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="")
ap.add_argument("--stride", type=int, default=7)
a = ap.parse_args()
pr = vp.load_config(2)
co = const_coeffs(pr.n_tri, pr.p)
sub = pr.txy[::a.stride]
exact = tri_potential_const(pr.vxy, pr.tri, sub)
rows = []
with vp.Evaluator(0) as ev:
    ev.set_mesh(pr.vxy, pr.tri)
    ev.set_far_method("fmm", 40)
    for eps, q in [(1e-8, 40), (1e-10, 40), (1e-12, 50), (1e-14, 50)]:
        ev.set_rules(vp.make_rules(q, eps=eps))
        ev.set_density(pr.p, co)
        for model in ("ball", "precise"):
            ev.set_near_model(model)
            u, st = ev.evaluate(sub)
            n = len(sub)
            r = {"eps": eps, "q": q, "model": model, "targets": n,
                 "c": (st["n_near_pairs"] + st["n_self"]) / n, "s_n": st["n_leaves"] / n,
                 "s_l": st["n_panels"] / max(st["n_self"], 1), "max_abs_err": float(np.abs(u - exact).max()),
                 "near_ms": st["t_near_ms"], "total_ms": st["t_total_ms"]}
            rows.append(r)
            print(json.dumps(r), flush=True)
        ev.set_near_model("precise")
if a.out:
    json.dump(rows, open(a.out, "w"), indent=1)
