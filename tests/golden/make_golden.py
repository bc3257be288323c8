"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Runs only in the build container (needs /root/reference and the shim
oracle/_ref/libvpref.so compiled from the reference headers by
`make ref`).  The outputs are small committed .npz/.json files; tests read
them on any machine (the GPU box has no /root/reference).

  koorn_ref.npz     koornwinder_eval(12, x, y) at 64 seeded points + corners
                    (koornwinder.hpp:123-126)
  gl_ref.npz        gauss_legendre(n), n = 1..24, 32 (gauss.hpp:17-46)
  quadtree_ref.npz  Quadtree::build(10^4 pts, m=8) + 100 query_rect results
                    (quadtree.hpp:24-62; rects lo=(x,y), hi=(x,y) order)
  ggq8_ref.json     the embedded_ggq8 table text of ggq.hpp:184-199 (data)
"""
import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import binding as ob  # noqa: E402

REF_GGQ = "/root/reference/proj/include/volpot/ggq.hpp"


def main():
    assert ob.ref() is not None, "build the shim first: make ref"
    rng = np.random.default_rng(1234)
    pts = []
    while len(pts) < 64:
        x, y = rng.random(2)
        if x + y <= 1:
            pts.append((x, y))
    pts += [(0.0, 0.0), (1.0, 0.0), (0.0, 1.0), (0.9999, 0.0), (0.3, 0.7), (0.5, 0.5)]
    pts = np.array(pts)
    vals = np.array([ob.ref_koornwinder(12, x, y) for x, y in pts])
    np.savez_compressed(os.path.join(HERE, "koorn_ref.npz"), pts=pts, vals=vals, order=12)

    ns = list(range(1, 25)) + [32]
    gl = {f"x{n}": ob.ref_gauss_legendre(n)[0] for n in ns}
    gl.update({f"w{n}": ob.ref_gauss_legendre(n)[1] for n in ns})
    np.savez_compressed(os.path.join(HERE, "gl_ref.npz"), ns=np.array(ns), **gl)

    rng = np.random.default_rng(2024)
    P = rng.random((10000, 2))
    rects, res, vis = [], [], []
    for _ in range(100):
        c, hw = rng.random(2), 0.1 * rng.random(2)
        r = (c[0] - hw[0], c[1] - hw[1], c[0] + hw[0], c[1] + hw[1])
        ids, v = ob.quadtree_query(P, 8, r, use_ref=True)
        rects.append(r)
        res.append(ids)
        vis.append(v)
    off = np.cumsum([0] + [len(r) for r in res])
    # points are regenerated from default_rng(2024) in the test; store a checksum
    np.savez_compressed(os.path.join(HERE, "quadtree_ref.npz"), pts_sum=P.sum(), rects=np.array(rects),
                        ids=np.concatenate(res).astype(np.int32), off=off, visited=np.array(vis))

    src = open(REF_GGQ).read()
    blk = src[src.index("embedded_ggq8() {"):]
    nums = [float(x) for x in re.findall(r"[0-9]\.[0-9]+e[-+][0-9]+", blk)][:18]
    with open(os.path.join(HERE, "ggq8_ref.json"), "w") as f:
        json.dump({"source": "ggq.hpp:184-199 embedded_ggq8()", "r": nums[:9], "w": nums[9:18]}, f,
                  indent=1)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
