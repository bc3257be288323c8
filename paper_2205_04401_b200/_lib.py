"""ctypes loader for libvp_b200.so (the C-ABI of include/vp.h + vp_setup.h).

The library is built in-tree by ``make`` (or ``__graft_entry__.build()``).
There is no fallback: if the shared object is missing, importing the
compute API raises, and on a machine without an sm_100 device every compute
entry point returns status 3 (device error).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# VP_B200_LIB overrides the library path (development builds / variant sweeps)
LIB_PATH = os.environ.get("VP_B200_LIB", os.path.join(_HERE, "libvp_b200.so"))

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_int64_p = ctypes.POINTER(ctypes.c_int64)


class VpRules(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_int), ("len_q", ctypes.c_int),
        ("far_x", c_double_p), ("far_y", c_double_p), ("far_w", c_double_p),
        ("n_n", ctypes.c_int), ("len_n", ctypes.c_int),
        ("near_x", c_double_p), ("near_y", c_double_p), ("near_w", c_double_p),
        ("n_l", ctypes.c_int), ("gl_x", c_double_p), ("gl_w", c_double_p),
        ("n_g", ctypes.c_int), ("ggq_r", c_double_p), ("ggq_w", c_double_p),
        ("eps", ctypes.c_double),
    ]


class VpStats(ctypes.Structure):
    _fields_ = [
        ("n_targets", ctypes.c_int64), ("n_outside", ctypes.c_int64),
        ("n_near_pairs", ctypes.c_int64), ("n_self", ctypes.c_int64),
        ("n_leaves", ctypes.c_int64), ("n_panels", ctypes.c_int64),
        ("n_rho_le1", ctypes.c_int64), ("n_degenerate", ctypes.c_int64),
        ("n_sources", ctypes.c_int64),
        ("max_depth", ctypes.c_int32), ("gpu_launches", ctypes.c_int32),
        ("t_list_ms", ctypes.c_double), ("t_far_ms", ctypes.c_double),
        ("t_near_ms", ctypes.c_double), ("t_self_ms", ctypes.c_double),
        ("t_total_ms", ctypes.c_double), ("t_sources_ms", ctypes.c_double),
        ("t_far_kernel_ms", ctypes.c_double),
        ("far_method", ctypes.c_int32), ("fmm_levels", ctypes.c_int32), ("fmm_outside", ctypes.c_int64),
        ("t_pair_ms", ctypes.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class VpsConfigInfo(ctypes.Structure):
    _fields_ = [
        ("n_vert", ctypes.c_int64), ("n_tri", ctypes.c_int64), ("n_tgt", ctypes.c_int64),
        ("p", ctypes.c_int), ("q", ctypes.c_int), ("density_kind", ctypes.c_int),
        ("n_params", ctypes.c_int), ("params", ctypes.c_double * 64), ("eps", ctypes.c_double),
        ("seed", ctypes.c_uint64), ("staggered", ctypes.c_int), ("pad", ctypes.c_int),
    ]


# (name, restype, argtypes) for every symbol declared in include/vp.h and vp_setup.h
_SIGS = [
    # vp.h
    ("vp_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    ("vp_destroy", None, [ctypes.c_void_p]),
    ("vp_last_error", ctypes.c_char_p, [ctypes.c_void_p]),
    ("vp_set_mesh", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, ctypes.c_int64, c_int32_p]),
    ("vp_set_curves", ctypes.c_int, [ctypes.c_void_p, c_int32_p, ctypes.c_int, ctypes.c_int64, c_double_p,
                                     c_double_p, c_double_p]),
    ("vp_set_rules", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(VpRules)]),
    ("vp_set_density", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_double_p]),
    ("vp_build_nearlist", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, c_int32_p,
                                         c_int64_p, c_int32_p, ctypes.c_int64, c_int64_p]),
    ("vp_evaluate", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, c_double_p,
                                   ctypes.POINTER(VpStats)]),
    ("vp_evaluate_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(VpStats)]),
    ("vp_evaluate_graph", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]),
    ("vp_graph_status", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(VpStats)]),
    ("vp_far_field", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, c_double_p]),
    ("vp_sources", ctypes.c_int, [ctypes.c_void_p, c_double_p, c_double_p, c_double_p]),
    ("vp_near_pairs", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, c_int32_p,
                                     c_double_p, c_double_p, c_int64_p]),
    ("vp_self_pairs", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, c_int32_p,
                                     c_double_p, c_double_p, c_int64_p]),
    ("vp_interp_coeffs", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_double_p, c_double_p, ctypes.c_int64,
                                        c_double_p, c_double_p, c_double_p]),
    ("vp_field_eval", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, ctypes.c_int64, c_int32_p,
                                     ctypes.c_int, c_double_p, ctypes.c_int64, c_double_p, c_double_p, c_int32_p,
                                     c_int64_p]),
    ("vp_set_near_model", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_double]),
    ("vp_set_near_cache", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64]),
    ("vp_set_far_method", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("vp_fmm_order_for", ctypes.c_int, [ctypes.c_double]),
    ("vp_set_fmm_tolerance", ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int]),
    ("vp_device_info", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("vp_shard_bounds", ctypes.c_int, [ctypes.c_int64, c_int64_p, ctypes.c_int, c_int64_p]),
    ("vp_shard_plan", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, ctypes.c_int, c_int32_p,
                                     c_int64_p, c_int64_p]),
    ("vp_nccl_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("vp_comm_init", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]),
    ("vp_gather", ctypes.c_int, [ctypes.c_void_p, c_int64_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    ("vp_allreduce_stats", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(VpStats)]),
    # vp_setup.h
    ("vps_koorn_size", ctypes.c_int, [ctypes.c_int]),
    ("vps_gauss_legendre", ctypes.c_int, [ctypes.c_int, c_double_p, c_double_p]),
    ("vps_gauss_jacobi10", ctypes.c_int, [ctypes.c_int, c_double_p, c_double_p]),
    ("vps_simplex_rule", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), c_double_p,
                                        c_double_p, c_double_p]),
    ("vps_quad_rule", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int), c_double_p,
                                     c_double_p, c_double_p]),
    ("vps_ggq", ctypes.c_int, [ctypes.c_int, c_double_p, c_double_p, c_double_p]),
    ("vps_circle_arc", ctypes.c_int, [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_int, c_double_p, c_double_p, c_double_p]),
    ("vps_curve_create", ctypes.c_int, [ctypes.c_int, c_double_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    ("vps_curve_destroy", None, [ctypes.c_void_p]),
    ("vps_curve_length", ctypes.c_double, [ctypes.c_void_p]),
    ("vps_curve_ccw", ctypes.c_int, [ctypes.c_void_p]),
    ("vps_curve_param", ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, c_double_p]),
    ("vps_curve_points", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, c_double_p, c_double_p,
                                        c_double_p]),
    ("vps_curve_closest", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_double_p, c_double_p, c_double_p]),
    ("vps_curve_segment", ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                         c_double_p, c_double_p, c_double_p]),
    ("vps_curve_last_error", ctypes.c_char_p, []),
    ("vps_lattice_nodes", ctypes.c_int, [ctypes.c_int, c_double_p, c_double_p]),
    ("vps_density_eval", ctypes.c_double, [ctypes.c_int, c_double_p, ctypes.c_int, ctypes.c_double,
                                           ctypes.c_double]),
    ("vps_project_density", ctypes.c_int, [ctypes.c_int64, c_double_p, ctypes.c_int64, c_int32_p,
                                           ctypes.c_int, ctypes.c_int, c_double_p, ctypes.c_int,
                                           c_double_p]),
    ("vps_config_info_get", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.POINTER(VpsConfigInfo)]),
    ("vps_config_fill", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, c_double_p,
                                       c_int32_p, c_double_p, c_double_p]),
    ("vps_last_error", ctypes.c_char_p, []),
]

SYMBOLS = [s[0] for s in _SIGS]

_lib = None


def lib():
    """Load libvp_b200.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
                "(there is no CPU fallback for the evaluator)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
