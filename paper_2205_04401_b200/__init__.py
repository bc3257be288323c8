"""B200-native evaluator for the 2-D log-kernel volume potential (arXiv 2205.04401 hot path).

Public API mirrors the reference's evaluation interface (see api.py); the
compute path is libvp_b200.so (sm_100a CUDA behind the C-ABI of include/vp.h).
"""
from .api import (  # noqa: F401
    DeviceError, Evaluator, NumericalError, Problem, Rules, UsageError, VolpotError, build_ggq,
    cn_lookup, config_info, density_eval, evaluate_field, fmm_eval, fmm_order_for, gauss_legendre, koorn_index,
    koorn_size, lattice_nodes, load_config, make_rules, project_density, quad_rule, simplex_rule,
    F_BUMPS, F_CONST, F_COSSIN, F_GAUSS, F_LINEAR, F_SQUARE, Curves, circle_arc, curve_boundary_of_disk, BoundaryCurve,
    curves_from_annotation, annotate_boundary, nccl_unique_id, shard_bounds, NCCL_ID_BYTES,
)
