"""One GPU's share of an N-way FMM evaluation (strong scaling of the FMM leg):
the far field of the first shard of vp_shard_plan (--targets shard) or of all
targets, on config 4 (or --config), at the default order or the order of
--eps.  Run under `ncu --metrics gpu__time_duration.sum` and summarise with
tools/launch_summary.py; VP_FMM_ALL_BOXES=1 gives the unrestricted downward
pass for comparison."""
import argparse, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04401_b200 as vp

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--targets", default="shard")
ap.add_argument("--eps", type=float, default=0.0)
a = ap.parse_args()
pr = vp.load_config(a.config)
with vp.Evaluator(0) as ev:
    ev.load(pr)
    if a.eps > 0:
        ev.set_fmm_tolerance(a.eps)
    else:
        ev.set_far_method("fmm")
    t = pr.txy
    if a.targets == "shard":
        order, bounds, cost = ev.shard_plan(pr.txy, a.world)
        t = np.ascontiguousarray(pr.txy[order][bounds[0]:bounds[1]])
    u = ev.far_field(t)
    print(f"config {a.config} targets {a.targets} n={len(t)} eps={a.eps} order={vp.fmm_order_for(a.eps) if a.eps > 0 else 31} "
          f"all_boxes={bool(os.environ.get('VP_FMM_ALL_BOXES'))} sum|u|={np.abs(u).sum():.6e}", flush=True)
