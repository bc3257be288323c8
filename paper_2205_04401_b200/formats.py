"""Text formats of the reference specification.

* Mesh file: header ``NV NE``; ``v x y bflag`` lines; then
  ``e i j k kind [opp curve s_a s_b]`` lines (kind 0 = straight, otherwise a
  curved element).  Written with 17 significant digits so
  a write/read round trip is bit-exact.
* Boundary-curve samples (curve.hpp:164-183): ``t x y dx dy`` rows.
* Node CSV: ``x,y,u`` per target.
* Sweep CSV (offload_sweep): ``Nf,TF,TN,TS,Ttot,c,sn``.
* Quadrature-rule table (rules.hpp:87-103): ``kind N len`` then ``x y w``.
"""
from __future__ import annotations

import io

import numpy as np


def write_mesh(path, vxy, tri, bflag=None, meta=None):
    """meta: optional rows (kind, opp, curve, s_a, s_b) per element; kind 0 =
    straight (annotate_boundary output)."""
    vxy = np.asarray(vxy, dtype=np.float64).reshape(-1, 2)
    tri = np.asarray(tri, dtype=np.int64).reshape(-1, 3)
    bflag = np.zeros(len(vxy), dtype=np.int64) if bflag is None else np.asarray(bflag, dtype=np.int64)
    with open(path, "w") as f:
        f.write(f"{len(vxy)} {len(tri)}\n")
        for (x, y), b in zip(vxy, bflag):
            f.write(f"v {x:.17g} {y:.17g} {int(b)}\n")
        for e, (i, j, k) in enumerate(tri):
            if meta is not None and int(meta[e][0]) != 0:
                kind, opp, cur, sa, sb = meta[e]
                f.write(f"e {i} {j} {k} {int(kind)} {int(opp)} {int(cur)} {float(sa):.17g} {float(sb):.17g}\n")
            else:
                f.write(f"e {i} {j} {k} 0\n")


def read_mesh(path, with_meta=False):
    """Returns (vxy, tri, bflag), plus the per-element curved-side metadata
    rows (kind, opp, curve, s_a, s_b) with with_meta=True; raises ValueError
    naming the violated invariant."""
    with open(path) as f:
        head = f.readline().split()
        if len(head) != 2:
            raise ValueError("mesh file: malformed header (expected `NV NE`)")
        nv, ne = int(head[0]), int(head[1])
        vxy = np.zeros((nv, 2))
        bflag = np.zeros(nv, dtype=np.int64)
        tri = np.zeros((ne, 3), dtype=np.int32)
        meta = np.zeros((ne, 5))
        for i in range(nv):
            t = f.readline().split()
            if len(t) < 4 or t[0] != "v":
                raise ValueError(f"mesh file: malformed vertex line {i}")
            vxy[i] = float(t[1]), float(t[2])
            bflag[i] = int(t[3])
        for i in range(ne):
            t = f.readline().split()
            if len(t) < 5 or t[0] != "e":
                raise ValueError(f"mesh file: malformed element line {i}")
            tri[i] = int(t[1]), int(t[2]), int(t[3])
            kind = int(t[4])
            if kind != 0:
                if not with_meta:
                    raise ValueError("mesh file: curved elements need read_mesh(..., with_meta=True)")
                if len(t) < 9:
                    raise ValueError(f"mesh file: curved element line {i} needs `opp curve s_a s_b`")
                opp = int(t[5])
                if opp < 0 or opp > 2:
                    raise ValueError(f"mesh file: opposite-vertex index of element {i} not in 0..2")
                meta[i] = kind, opp, int(t[6]), float(t[7]), float(t[8])
    if tri.size and (tri.min() < 0 or tri.max() >= nv):
        raise ValueError("mesh file: element vertex index out of range")
    return (vxy, tri, bflag, meta) if with_meta else (vxy, tri, bflag)


def read_curve_samples(path_or_buf):
    """Hermite boundary-curve samples, one `t x y dx dy` row per line, `#`
    comments (curve.hpp:164-183)."""
    text = path_or_buf.read() if hasattr(path_or_buf, "read") else open(path_or_buf).read()
    rows = []
    for line in text.splitlines():
        if not line.strip() or line.lstrip().startswith("#"):
            continue
        tok = line.split()
        if len(tok) < 5:
            raise ValueError("curve file: expected `t x y dx dy` per line")
        rows.append([float(v) for v in tok[:5]])
    return np.array(rows).reshape(-1, 5)


def write_nodes_csv(path, txy, u):
    txy = np.asarray(txy, dtype=np.float64).reshape(-1, 2)
    with open(path, "w") as f:
        f.write("x,y,u\n")
        for (x, y), v in zip(txy, np.asarray(u, dtype=np.float64)):
            f.write(f"{x:.17g},{y:.17g},{v:.17g}\n")


def write_sweep_csv(path, rows):
    """rows: dicts with Nf, TF, TN, TS, Ttot, c, sn (SPEC.md offload_sweep)."""
    with open(path, "w") as f:
        f.write("Nf,TF,TN,TS,Ttot,c,sn\n")
        for r in rows:
            f.write(f"{r['Nf']},{r['TF']:.6g},{r['TN']:.6g},{r['TS']:.6g},{r['Ttot']:.6g},{r['c']:.6g},{r['sn']:.6g}\n")


def write_rule(path_or_buf, kind, order, x, y, w):
    buf = io.StringIO()
    buf.write(f"{kind} {order} {len(x)}\n")
    for a, b, c in zip(x, y, w):
        buf.write(f"{a:.17g} {b:.17g} {c:.17g}\n")
    text = buf.getvalue()
    if hasattr(path_or_buf, "write"):
        path_or_buf.write(text)
    else:
        with open(path_or_buf, "w") as f:
            f.write(text)


def read_rule(path_or_buf):
    """Parse a rule table; raises ValueError with the reference's messages
    (rules.hpp:88-103)."""
    text = path_or_buf.read() if hasattr(path_or_buf, "read") else open(path_or_buf).read()
    tok = text.split()
    if len(tok) < 3:
        raise ValueError("rule table: malformed header (expected `kind N len`)")
    kind, order, n = tok[0], int(tok[1]), int(tok[2])
    if kind not in ("X-G", "XG", "xiao-gimbutas", "V-R", "VR", "vioreanu-rokhlin"):
        raise ValueError(f"rule table: unknown kind `{kind}`")
    vals = tok[3:]
    if len(vals) < 3 * n:
        raise ValueError("rule table: truncated node list")
    a = np.array([float(v) for v in vals[:3 * n]]).reshape(n, 3)
    return kind, order, a[:, 0], a[:, 1], a[:, 2]
