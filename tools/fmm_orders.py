import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2205_04401_b200 as vp
def rel(a, b): return float(np.abs(a - b).max() / np.abs(b).max())
for cfg, stride in ((1,1),(2,1),(3,10),(4,150)):
    pr = vp.load_config(cfg)
    sub = pr.txy[::stride]
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ud = ev.far_field(sub)
        for p in (27, 31, 36):
            ev.set_far_method("fmm", p)
            uf = ev.far_field(sub)
            print(f"cfg{cfg} p={p}: far rel err {rel(uf, ud):.2e}", flush=True)
