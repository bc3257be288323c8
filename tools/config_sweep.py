"""Per-configuration statistics on the GPU (BASELINE configs 3, 4 and the
config-5 far-order sweep q in {p+2, 2p, 3p}).

Full-size meshes, densities and sources; targets are a deterministic
subsample (every k-th target), so the far work per target is exact and the
per-target rates extrapolate linearly to the full target set.  Prints one
JSON line per run and writes profiles/r01_config_sweep.json.

  python tools/config_sweep.py [--stride 100] [--configs 3,4,5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04401_b200 as vp  # noqa: E402


def run(cfg, q, stride, ev=None):
    t0 = time.time()
    pr = vp.load_config(cfg, q)
    gen_s = time.time() - t0
    sub = pr.txy[::stride]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ev.evaluate(sub[:2048])  # warm-up (lazy module loading, clocks)
        ev.evaluate(sub)
        u, st = ev.evaluate(sub)
    n = len(sub)
    T = pr.n_tgt
    out = {
        "config": cfg, "q": pr.q, "p": pr.p, "n_tri": pr.n_tri, "targets_full": T,
        "targets_sampled": n, "stride": stride, "sources": st["n_sources"],
        "far_pairs_full": T * st["n_sources"],
        "near_pairs_per_target": st["n_near_pairs"] / n,
        "c_corrections_per_target": (st["n_near_pairs"] + st["n_self"]) / n,
        "s_n_leaves_per_target": st["n_leaves"] / n,
        "s_l_panels_per_self": st["n_panels"] / max(st["n_self"], 1),
        "outside": st["n_outside"], "max_depth": st["max_depth"], "rho_le1": st["n_rho_le1"],
        "ms_sample": {k: st[k] for k in ("t_list_ms", "t_far_ms", "t_near_ms", "t_self_ms", "t_total_ms")},
        "extrapolated_full_s": {k: st[k] * 1e-3 * T / n for k in ("t_list_ms", "t_far_ms", "t_near_ms",
                                                                   "t_self_ms", "t_total_ms")},
        "targets_per_s": n / (st["t_total_ms"] * 1e-3),
        "far_pairs_per_s": n * st["n_sources"] / (st["t_far_ms"] * 1e-3),
        "u_finite": bool(np.isfinite(u).all()), "generate_s": gen_s,
    }
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stride", type=int, default=100)
    ap.add_argument("--configs", default="3,4,5")
    ap.add_argument("--out", default="profiles/r01_config_sweep.json")
    a = ap.parse_args()
    res = []
    for c in [int(x) for x in a.configs.split(",")]:
        if c == 5:
            for q in (10, 16, 24):
                res.append(run(5, q, a.stride))
        else:
            res.append(run(c, 0, a.stride))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
