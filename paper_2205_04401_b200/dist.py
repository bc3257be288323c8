"""Multi-GPU plumbing: targets are sharded, mesh + density replicated, and
the only collective is the gather of u (BASELINE.json north_star; SURVEY.md
§8(e)).  One process per GPU; torch.distributed carries the collective
(NCCL on B200 boxes, gloo in the CPU tests).

Per-target results are independent and computed by fixed-order reductions,
so u(t) is bit-identical whatever the shard layout (the invariant tested in
tests/test_multirank.py and tests/test_gpu_parity.py).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n: int, rank: int, world: int):
    """Contiguous, equal-count (+-1) range [lo, hi) of n targets for `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("shard_bounds: need 0 <= rank < world")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def padded_shard(n: int, world: int) -> int:
    """Per-rank length of the padded equal shards used by all_gather."""
    return (n + world - 1) // world


def gather_potentials(u_local, n_total: int, rank: int, world: int, group=None):
    """All-gather per-rank shards of u (torch tensors, any device) into the
    full vector on every rank.  Shards are padded to equal length so one
    all_gather_into_tensor moves everything (NCCL over NVLink on B200)."""
    import torch
    import torch.distributed as dist

    m = padded_shard(n_total, world)
    lo, hi = shard_bounds(n_total, rank, world)
    buf = torch.zeros(m, dtype=u_local.dtype, device=u_local.device)
    buf[: hi - lo] = u_local
    out = torch.empty(m * world, dtype=u_local.dtype, device=u_local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = []
    for r in range(world):
        a, b = shard_bounds(n_total, r, world)
        parts.append(out[r * m: r * m + (b - a)])
    return torch.cat(parts)


def morton_order(txy) -> np.ndarray:
    """Permutation sorting targets along a Morton (Z-order) curve so that
    contiguous shards are spatially compact (near/self work stays local)."""
    t = np.asarray(txy, dtype=np.float64).reshape(-1, 2)
    lo, hi = t.min(0), t.max(0)
    span = np.where(hi > lo, hi - lo, 1.0)
    q = np.minimum(((t - lo) / span * 65535.0).astype(np.uint64), 65535)

    def spread(v):
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
        return v

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1))
    return np.argsort(code, kind="stable")
