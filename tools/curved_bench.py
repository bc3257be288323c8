"""Curved-disk timing: config 2 with its 256 boundary triangles curved on the
exact circle vs the same mesh straight."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2205_04401_b200 as vp  # noqa: E402

KEYS = ("t_total_ms", "t_list_ms", "t_far_ms", "t_near_ms", "t_self_ms", "n_leaves", "n_panels", "n_self")


def main():
    pr = vp.load_config(2)
    tri, cv = vp.curve_boundary_of_disk(pr.vxy, pr.tri)
    co = vp.project_density(pr.vxy, tri, pr.p, vp.F_GAUSS, [0.2, -0.1, 3.0])
    ev = vp.Evaluator(0)
    ev.set_mesh(pr.vxy, tri)
    ev.set_curves(cv)
    ev.set_rules(pr.rules)
    ev.set_density(pr.p, co)
    out = {}
    for name in ("curved", "straight"):
        best = None
        for _ in range(5):
            _, st = ev.evaluate(pr.txy)
            if best is None or st["t_total_ms"] < best["t_total_ms"]:
                best = st
        out[name] = {k: best[k] for k in KEYS}
        ev.set_curves(None)
    out["curved_elements"] = int((cv.curve_id >= 0).sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
