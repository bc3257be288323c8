"""One GPU's share of an N-way strong-scaling run of the full-size legs, on ONE
GPU: evaluates the whole config-4 target set and then single shards of
vp_shard_plan (the work rank r would do), with far method none (pair stage)
and fmm.  The ratio t_full / (N * max_r t_shard) is what the sharding itself
costs (per-rank work that does not shrink with N, imbalance of the plan); the
NCCL gather of u (N * 8 B per target) is not in it.  A projection from one
GPU's share, not a multi-GPU measurement.

  python tools/shard_share.py [--config 4] [--world 8] [--ranks 0,3,7] OUT.json"""
import argparse, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04401_b200 as vp

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--ranks", default="0,3,7")
a = ap.parse_args()
ranks = [int(r) for r in a.ranks.split(",")]
pr = vp.load_config(a.config)
KEYS = ("t_total_ms", "t_list_ms", "t_far_ms", "t_pair_ms", "t_near_ms", "t_self_ms")
doc = {"config": a.config, "world": a.world, "targets": int(pr.n_tgt), "legs": {}}
with vp.Evaluator(0) as ev:
    ev.load(pr)
    for far in ("none", "fmm"):
        ev.set_far_method(far)
        order, bounds, cost = ev.shard_plan(pr.txy, a.world)

        def run(t):
            ev.evaluate(t)
            best = None
            for _ in range(3):
                _, st = ev.evaluate(t)
                if best is None or st["t_total_ms"] < best["t_total_ms"]:
                    best = st
            return {k: best[k] for k in KEYS}

        full = run(pr.txy)
        shards = {}
        for r in ranks:
            t = np.ascontiguousarray(pr.txy[order[bounds[r]:bounds[r + 1]]])
            shards[r] = dict(run(t), targets=int(len(t)), plan_cost=int(cost[r]))
        worst = max(s["t_total_ms"] for s in shards.values())
        leg = {"full": full, "shards": shards, "ideal_ms": full["t_total_ms"] / a.world,
               "share_efficiency": full["t_total_ms"] / (a.world * worst)}
        doc["legs"][far] = leg
        print(far, json.dumps(leg), flush=True)
json.dump(doc, open(a.out, "w"), indent=1)
