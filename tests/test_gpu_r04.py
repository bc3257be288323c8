"""GPU parity, round 2 (last session): the FMM order chosen from a far-field
tolerance and the downward pass restricted to the boxes that
hold targets (a shard pays for its own part of the tree).

The far field of the FMM is compared with the library's own direct sum, which
test_gpu_parity.py holds against the CPU oracle."""
import numpy as np
import pytest

import paper_2205_04401_b200 as vp

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("cfg,stride", [(2, 3), (3, 40)])
def test_fmm_tolerance_bounds_the_far_field_error(cfg, stride):
    pr = vp.load_config(cfg)
    sub = np.ascontiguousarray(pr.txy[::stride])
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        ud = ev.far_field(sub)
        last = None
        for eps in (1e-3, 1e-5, 1e-7, 1e-9, 1e-11, 1e-13):
            ev.set_fmm_tolerance(eps)
            err = rel(ev.far_field(sub), ud)
            assert err <= eps, f"config {cfg}: eps_fmm {eps:g} (order {vp.fmm_order_for(eps)}) gave {err:.2e}"
            assert last is None or err <= 4 * last  # tighter tolerance, no worse result
            last = err
        with pytest.raises(vp.UsageError):
            ev.set_fmm_tolerance(0.0)
        with pytest.raises(vp.UsageError):
            ev.set_fmm_tolerance(2.0)


def test_fmm_shard_equals_whole_bitwise():
    """The boxes the downward pass skips for a shard do not change its u:
    a spatially compact shard (few active boxes) and scattered targets
    reproduce the all-targets evaluation bit for bit, for the one-lane-per-
    coefficient kernel (order 31, 19) and the generic one (order 22)."""
    pr = vp.load_config(2)
    t = pr.txy
    compact = np.flatnonzero((t[:, 0] > 0.1) & (t[:, 0] < 0.3) & (t[:, 1] > -0.2) & (t[:, 1] < 0.0))
    scattered = np.arange(0, len(t), 97)
    assert compact.size > 500
    with vp.Evaluator(0) as ev:
        ev.load(pr)
        for order in (31, 19, 22):
            ev.set_far_method("fmm", order)
            u_all, _ = ev.evaluate(t)
            for idx in (compact, scattered):
                u_s, st = ev.evaluate(np.ascontiguousarray(t[idx]))
                assert st["far_method"] == 1
                assert np.array_equal(u_s, u_all[idx]), f"order {order}"
