"""Near-stage device time against the near-leaf cache depth (config 2 by
default): python tools/cache_depth.py [config] [depths, e.g. 2,3,4]  (GPU box)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_04401_b200 as vp  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pr = vp.load_config(cfg)
ev = vp.Evaluator(0).load(pr)
ev.set_far_method("fmm")  # the near stage is what is measured
depths = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [-1, 1, 2, 3, 4, 5]
d_txy = torch.from_numpy(pr.txy).cuda()
d_u = torch.empty(pr.n_tgt, dtype=torch.float64, device="cuda")
ref = None
for D in depths:
    ev.set_near_cache(D, 64 << 30)
    for _ in range(3):
        ev.evaluate_device(pr.n_tgt, d_txy.data_ptr(), d_u.data_ptr())
    torch.cuda.synchronize()
    sts = [ev.evaluate_device(pr.n_tgt, d_txy.data_ptr(), d_u.data_ptr()) for _ in range(5)]
    torch.cuda.synchronize()
    u = d_u.cpu().numpy()
    if ref is None:
        ref = u.copy()
    print(f"D={D:2d} near {np.mean([s['t_near_ms'] for s in sts]):.3f} ms  self {np.mean([s['t_self_ms'] for s in sts]):.3f}"
          f"  total {np.mean([s['t_total_ms'] for s in sts]):.2f}  max|du|/max|u| {np.abs(u - ref).max() / np.abs(ref).max():.2e}",
          flush=True)
