"""Full-size evaluation of a BASELINE config on one GPU (FMM far field by default),
with parity against the CPU oracle on a target sample.

  python tools/full_config.py --config 4 [--far fmm] [--check 400]
"""
import argparse, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04401_b200 as vp  # noqa: E402
from oracle.binding import Oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--q", type=int, default=0)
ap.add_argument("--far", default="fmm")
ap.add_argument("--check", type=int, default=400)
ap.add_argument("--out", default="")
ap.add_argument("--cache-depth", type=int, default=-2, help="near cache max depth (-2: library default)")
ap.add_argument("--cache-gb", type=float, default=0.0, help="near cache byte budget in GB (0: default)")
a = ap.parse_args()
t0 = time.time()
pr = vp.load_config(a.config, a.q)
gen = time.time() - t0
with vp.Evaluator(0) as ev:
    ev.load(pr)
    ev.set_far_method(a.far)
    if a.cache_depth != -2 or a.cache_gb > 0:
        ev.set_near_cache(a.cache_depth if a.cache_depth != -2 else 3, int(a.cache_gb * (1 << 30)))
    ev.evaluate(pr.txy)  # warm-up at full size: device buffers allocated outside the timed pass
    t1 = time.time()
    u, st = ev.evaluate(pr.txy)
    wall = time.time() - t1
err, ocpu = None, float("nan")
if a.check > 0:
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(pr.n_tgt, a.check, replace=False))
    t2 = time.time()
    u_o, _, sto = Oracle.from_problem(pr).evaluate(pr.txy[idx])
    ocpu = time.time() - t2
    err = float(np.abs(u[idx] - u_o).max() / np.abs(u_o).max())
out = {"config": a.config, "q": pr.q, "far": a.far, "n_tri": pr.n_tri, "targets": pr.n_tgt,
       "sources": st["n_sources"], "near_pairs": st["n_near_pairs"], "leaves": st["n_leaves"],
       "panels": st["n_panels"], "outside": st["n_outside"], "fmm_levels": st["fmm_levels"],
       "device_ms": {k: st[k] for k in ("t_list_ms", "t_sources_ms", "t_far_ms", "t_near_ms", "t_self_ms", "t_pair_ms", "t_total_ms")},
       "wall_s": wall, "targets_per_s_device": pr.n_tgt / (st["t_total_ms"] * 1e-3),
       "parity_sample": a.check, "u_rel_err_vs_oracle": err, "oracle_cpu_s": ocpu,
       "oracle_targets_per_s_cpu": (a.check / ocpu) if a.check > 0 else None, "generate_s": gen}
print(json.dumps(out), flush=True)
if a.out:
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
