"""Far-field error of the FMM against the direct sum by expansion order, on
configs 1-3 (and a strided config 4): the calibration of vp_fmm_order_for
(eps_fmm -> order).  Writes JSON to argv[1]."""
import json
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2205_04401_b200 as vp


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


out = {}
orders = (4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26, 28, 31, 34, 38, 42)
for cfg, stride in ((1, 1), (2, 1), (3, 10), (4, 150)):
    pr = vp.load_config(cfg)
    sub = pr.txy[::stride]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ud = ev.far_field(sub)
        row = {}
        for p in orders:
            ev.set_far_method("fmm", p)
            row[p] = rel(ev.far_field(sub), ud)
        out[f"config{cfg}"] = row
        print(cfg, " ".join(f"{p}:{e:.1e}" for p, e in row.items()), flush=True)
json.dump(out, open(sys.argv[1], "w"), indent=1)
