"""Multi-rank host logic on CPU with the gloo backend (world_size 2).

On B200 boxes each rank drives its own GPU and the collective is NCCL; the
sharding and gather code is the same.  Per-target results are independent,
so the gathered u must be bit-identical to the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2205_04401_b200.dist import gather_potentials, morton_order, padded_shard, shard_bounds


def test_shard_bounds_partition():
    for n in (0, 1, 7, 100, 184320):
        for world in (1, 2, 3, 4, 8):
            b = [shard_bounds(n, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1 and max(sizes) <= padded_shard(n, world)


def test_morton_order_is_permutation():
    t = np.random.default_rng(0).random((1000, 2))
    o = morton_order(t)
    assert np.array_equal(np.sort(o), np.arange(1000))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2205_04401_b200 as vp
    from oracle.binding import Oracle
    pr = vp.load_config(1)
    txy = pr.txy[::3]
    lo, hi = shard_bounds(len(txy), rank, world)
    u, _, _ = Oracle.from_problem(pr).evaluate(txy[lo:hi], nthreads=2)
    full = gather_potentials(torch.from_numpy(u), len(txy), rank, world)
    if rank == 0:
        np.save(out, full.numpy())
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_gloo_two_rank_gather_is_bit_identical(tmp_path):
    out = str(tmp_path / "u.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    import paper_2205_04401_b200 as vp
    from oracle.binding import Oracle
    pr = vp.load_config(1)
    u1, _, _ = Oracle.from_problem(pr).evaluate(pr.txy[::3], nthreads=2)
    assert np.array_equal(np.load(out), u1)


def test_bench_shards_partition_the_job():
    """bench.py's strong-scaling job: config 4's targets in Morton order, every
    256th; N contiguous shards cover it exactly once at every N, and bench's
    Morton order is the product's (dist.morton_order)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import paper_2205_04401_b200 as vp
    from paper_2205_04401_b200.dist import morton_order, shard_bounds
    pr = vp.load_config(2, with_rules=False)
    assert np.array_equal(bench.morton_order(pr.txy), morton_order(pr.txy))
    assert bench.auto_stride(29360128, 51380224) == 256
    assert bench.auto_stride(184320, 331776) == 1
    sub = bench.headline_targets(pr.txy, 8)
    assert np.array_equal(sub, pr.txy[morton_order(pr.txy)[::8]])
    for world in (1, 2, 4, 8):
        parts = [bench.shard_bounds(len(sub), r, world) for r in range(world)]
        assert parts == [shard_bounds(len(sub), r, world) for r in range(world)]
        assert parts[0][0] == 0 and parts[-1][1] == len(sub)
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1


def test_bench_config_identical_across_arms():
    """Both arms print the same config dict for the same arguments."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    a = bench.workload_config(4, 1048576, 6, 12, 1e-12, 0, 29360128, 51380224, 256, 114688, 1)
    b = bench.workload_config(4, 1048576, 6, 12, 1e-12, 0, 29360128, 51380224, 256, 114688, 1)
    assert a == b and a["workload"] == "config4" and a["targets"] == 114688


def test_shard_bounds_host():
    """vp_shard_bounds (host only): contiguous cover, balanced to one item's
    cost, equal to a numpy restatement of its definition."""
    import paper_2205_04401_b200 as vp
    rng = np.random.default_rng(5)
    for n, world in [(0, 3), (1, 4), (10, 3), (1000, 8), (12345, 7)]:
        cost = rng.integers(0, 1000, size=n).astype(np.int64)
        b = vp.shard_bounds(cost, world)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        P = np.concatenate([[0], np.cumsum(cost)])
        ref = [0] + [int(np.searchsorted(P * world >= r * P[-1], True)) if False else
                     int(np.argmax(P * world >= r * P[-1])) for r in range(1, world)] + [n]
        assert list(b) == ref
        if n:
            per = [P[b[r + 1]] - P[b[r]] for r in range(world)]
            assert max(per) <= P[-1] / world + cost.max()
    with pytest.raises(vp.UsageError):
        vp.shard_bounds([1, -1], 2)
