"""FMM far field vs the direct far sum (development check; tests/ hold the gates)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2205_04401_b200 as vp


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def run(cfg, stride, orders=(24, 32, 40, 48)):
    pr = vp.load_config(cfg)
    sub = pr.txy[::stride]
    sub = np.vstack([sub, [[5.0, 5.0], [-3.0, 0.1]]])  # two targets outside the root box
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ud = ev.far_field(sub)
        u_dir, st_d = ev.evaluate(sub)
        for p in orders:
            ev.set_far_method("fmm", p)
            uf = ev.far_field(sub)
            uf = ev.far_field(sub)
            t = time.time(); u_f, st = ev.evaluate(sub); dt = time.time() - t
            print(f"cfg{cfg} T={len(sub)} p={p}: far rel err {rel(uf, ud):.2e}  u rel err {rel(u_f, u_dir):.2e}  "
                  f"far {st['t_far_ms']:.2f} ms (direct {st_d['t_far_ms']:.2f})  levels {st['fmm_levels']} "
                  f"outside {st['fmm_outside']}  total {st['t_total_ms']:.2f} ms", flush=True)
        ev.set_far_method("direct")


run(1, 1)
run(2, 1)
run(3, 20)
run(4, 200, orders=(40, 48))
