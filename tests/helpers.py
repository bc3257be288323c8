"""Shared test helpers: analytic potentials and small meshes."""
import numpy as np


def tri_potential_const(vxy, tri, x):
    """(1/2pi) sum_T int_T log|x-y| dA(y) for f = 1, closed form.

    Divergence theorem with Phi = r^2 (log r - 1)/4 (Laplacian log r):
    int_T log r dA = sum_edges h_e int_e (log r / 2 - 1/4) ds, h_e the signed
    distance from x to the edge line along the outward normal.
    """
    x = np.asarray(x, float).reshape(-1, 2)
    u = np.zeros(len(x))
    for t in np.asarray(tri).reshape(-1, 3):
        for k in range(3):
            P = vxy[t[k]]
            Q = vxy[t[(k + 1) % 3]]
            d = Q - P
            ln = np.hypot(*d)
            tau = d / ln
            n = np.array([tau[1], -tau[0]])
            h = (P - x) @ n
            s0 = (x - P) @ tau

            def G(a):
                with np.errstate(divide="ignore", invalid="ignore"):
                    lg = np.where(a * a + h * h > 0, np.log(a * a + h * h), 0.0)
                    at = np.where(h != 0, h / 2 * np.arctan(a / np.where(h != 0, h, 1)), 0.0)
                return a / 4 * lg - 0.75 * a + at

            u += h * (G(ln - s0) - G(-s0))
    return u / (2 * np.pi)


def const_coeffs(n_tri, p, value=1.0):
    c = np.zeros((n_tri, (p + 1) * (p + 2) // 2))
    c[:, 0] = value / np.sqrt(2.0)  # K_00 = sqrt(2)
    return c


def small_mesh():
    """Two triangles forming the unit square (diagonal (0,0)-(1,1))."""
    vxy = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    tri = np.array([[0, 1, 3], [0, 3, 2]], dtype=np.int32)
    return vxy, tri


def brute_nearlist(vxy, tri, models_two_a, all_near, txy):
    """Independent list oracle: direct scan of every element with the same
    IEEE operation order as the specified predicate (numpy, no FMA)."""
    E = len(tri)
    S, lists = [], []
    x0 = vxy[tri[:, 0]]
    e1 = vxy[tri[:, 1]] - x0
    e2 = vxy[tri[:, 2]] - x0
    det = e1[:, 0] * e2[:, 1] - e2[:, 0] * e1[:, 1]
    i00, i01 = e2[:, 1] / det, -e2[:, 0] / det
    i10, i11 = -e1[:, 1] / det, e1[:, 0] / det
    for tx, ty in txy:
        dx, dy = tx - x0[:, 0], ty - x0[:, 1]
        xi = i00 * dx + i01 * dy
        eta = i10 * dx + i11 * dy
        l0 = (1.0 - xi) - eta
        inside = (xi >= -1e-12) & (eta >= -1e-12) & (l0 >= -1e-12)
        s = int(np.argmax(inside)) if inside.any() else -1
        d = [np.sqrt((tx - vxy[tri[:, k], 0]) ** 2 + (ty - vxy[tri[:, k], 1]) ** 2) for k in range(3)]
        near = ((d[0] + d[1] < models_two_a[:, 0]) | (d[1] + d[2] < models_two_a[:, 1])
                | (d[2] + d[0] < models_two_a[:, 2]) | all_near)
        if s >= 0:
            near[s] = False
        S.append(s)
        lists.append(np.nonzero(near)[0])
    off = np.cumsum([0] + [len(x) for x in lists])
    ids = np.concatenate(lists) if lists else np.zeros(0, int)
    return np.array(S), off, ids
