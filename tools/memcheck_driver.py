"""Small end-to-end run for compute-sanitizer: every kernel of both far
methods, the near cache, interpolation and field evaluation on config 1."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2205_04401_b200 as vp
pr = vp.load_config(1)
with vp.Evaluator(0) as ev:
    ev.load(pr)
    sub = np.vstack([pr.txy[::5], [[3.0, 3.0]]])
    u, _ = ev.evaluate(sub)
    ev.set_far_method("fmm", 24)
    u2, _ = ev.evaluate(sub)
    ev.set_near_model("ball")
    u3, _ = ev.evaluate(sub)
    ev.set_near_model("precise")
    ev.far_field(sub)
    s, off, ids = ev.build_nearlist(sub)
    ev.near_pairs(sub[:10], np.zeros(10, dtype=np.int32) + 3)
    ev.self_pairs(pr.txy[:10], np.arange(10) // 15)
    lx, ly = vp.lattice_nodes(pr.p)
    co, _ = ev.interp_coeffs(pr.p, lx, ly, np.ones((pr.n_tri, vp.koorn_size(pr.p))))
    ev.field_eval(pr.vxy, pr.tri, pr.p, co, sub, allow_outside=True)
print("memcheck driver ok", float(np.abs(u - u2).max()))
