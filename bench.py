#!/usr/bin/env python
"""Benchmark of the volume-potential hot path (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W --config 4 --impl b200|reference]

Workload (default BASELINE config 4, the largest single-GPU configuration
and north_star's 1/2/4/8-GPU case: unit square, 1,048,576 jittered
triangles, p = 6, q = 12, 29,360,128 staggered targets, 34,603,008 far
sources: 33 per triangle, the symmetric order-12 rule).  One step = one full evaluation pass through the library (K3
near-field lists, K1 strengths, K2 direct far sum, K4 near pairs, K5 self
pairs, assembly) over one batch of targets:

  * headline `value` -- the direct far path (north_star part 3) over a
    deterministic target subset: the config's targets in Morton order, every
    `stride`-th (config 4: every 128th, 229,376 targets), each with its full
    34.6 M-source far field (SURVEY.md §7/§8(d) allow a stated fixed subset;
    a full direct config-4 step is about 13 minutes).  Strong scaling: the
    job is that subset whatever N, cut into N contiguous Morton shards.
  * `pair_stage` -- the near/self corrections of ALL the config's targets
    (far method "none"): BASELINE's second metric, near-field pair
    integrals/s, and the pair-stage FP64 roofline.
  * `alt_far_method` -- the full evaluation of ALL targets with the FMM far
    field.

Before timing, rank 0 checks its own u on a 512-target sample of the subset
against the CPU oracle (built from the oracle's own generators, no product
code), which doubles as `cpu_baseline`.

--impl reference times the CPU oracle (oracle/, a restatement of the
reference's specified path; the reference has no implementation of it,
SURVEY.md §0.1) on all host cores, over bounded slices of the same target
subset, with the same config dict; it loads only oracle/ libraries.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# Algorithmic work of one far pair as formulated on B200:
# dx, dy (2 DADD), r^2 (DMUL + DFMA), log r^2 (5 DFMA: t, 3-term polynomial
# on the 10-bit table, exponent), accumulate (1 DFMA) = 10 FP64 operations =
# 7 FMA (2 flops) + 3 add/mul (1 flop) = 17 flops.  This supersedes SURVEY.md
# §8(d)'s frozen 51 flops/pair, which counted libdevice's log (33 FP64
# instructions); the ncu SASS counters of K2 must agree (flop_per_pair_ncu).
FAR_FLOP_PER_PAIR = 17
SURVEY_FAR_FLOP_PER_PAIR = 51
# SURVEY.md §8(d) frozen algorithmic work of the near and self pairs (a direct
# implementation: Koornwinder evaluation at every leaf / panel node)
SURVEY_KP = {4: 117, 6: 226, 8: 371, 12: 769}
CHECK_SAMPLE = 512      # oracle check / cpu_baseline targets (rank 0, before timing)
CHECK_TOL = 1e-11       # north_star: potentials within 1e-11 relative max-norm
DIRECT_STEP_PAIRS = 6e12  # target subset stride: about 5 s of K2 per step


def survey_near_self_flops(st, p, len_q, len_n=49, n_l=16, n_g1=9):
    kp = SURVEY_KP.get(p)
    if kp is None:
        return None
    m2 = (p + 1) * (p + 2)
    return (st["n_leaves"] * len_n * (m2 + 60) + st["n_near_pairs"] * len_q * 51
            + st["n_panels"] * n_l * (60 + n_g1 * (kp + m2 + 10)) + st["n_self"] * len_q * 51)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--q", type=int, default=0, help="far order override (config 5 sweep)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--stride", type=int, default=0,
                    help="headline target subset: every stride-th target in Morton order (0: auto)")
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--mode", choices=["all", "pairs"], default="all",
                    help="pairs: only the full-size pair stage (for tools/fp64_flops.py)")
    ap.add_argument("--no-fmm", action="store_true", help="skip the full-size FMM measurement")
    ap.add_argument("--no-pairs", action="store_true", help="skip the full-size pair-stage measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the oracle check / cpu_baseline")
    ap.add_argument("--ref-chunk", type=int, default=0, help="--impl reference: targets per step (0: auto)")
    ap.add_argument("--near-cache-depth", type=int, default=3, help="vp_set_near_cache max depth")
    ap.add_argument("--near-cache-gb", type=float, default=0, help="vp_set_near_cache byte budget (0: library default)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------
# workload definition, shared by both arms (no product code: the reference
# arm must not load libvp_b200.so)

def morton_order(txy) -> np.ndarray:
    """Z-order permutation of the targets (same as paper_2205_04401_b200.dist.
    morton_order; tests/test_bench.py checks they agree)."""
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


def auto_stride(n_tgt, n_src):
    """The power of two nearest (in log) to T*S / 6e12, at least 1: about
    5 s of direct far sum per step on one B200."""
    r = n_tgt * n_src / DIRECT_STEP_PAIRS
    return 1 if r < 1.5 else 2 ** int(round(np.log2(r)))


def shard_bounds(n, rank, world):
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def headline_targets(txy, stride):
    """The headline target subset: Morton order, every stride-th."""
    order = morton_order(txy)
    return np.ascontiguousarray(txy[order[::stride]])


def workload_config(cfg, n_tri, p, q, eps, seed, n_tgt, n_src, stride, n_sub, world):
    """The config dict both arms print (identical for the same arguments)."""
    return {"workload": f"config{cfg}", "n_tri": int(n_tri), "p": int(p), "q": int(q), "eps": float(eps),
            "seed": int(seed), "targets_full": int(n_tgt), "sources": int(n_src),
            "target_subset": (f"every {stride}th target in Morton order" if stride > 1 else "all targets"),
            "targets": int(n_sub), "far_method": "direct",
            "l2": "inputs > L2 (sources %.2f GB) and a 256 MB L2 flush between timed steps" % (24 * n_src / 1e9),
            "parallelism": f"targets sharded over {world} GPU(s), Morton-contiguous (strong scaling); "
                           "mesh + density replicated; u gathered over NCCL"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.window = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def wait_first(self, timeout=10.0):
        """NVML start-up can stall CUDA calls of this process, so the sampler
        starts before the warm-up and timing begins after its first sample."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.05)

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=1)
        if self.window is not None:
            a, b = self.window
            inside = [r for r in self.rows if a - 0.1 <= r[0] <= b + 0.1]
            self.rows = inside or self.rows[-1:]
        self.rows = [r[1] for r in self.rows]
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6
                          for i in range(4) if r[2 + i].lower().startswith("active")})
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": reasons, "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def fp64_peak():
    """FP64 roofline denominator: MEASURED_PEAKS.json has no FP64 entry, so
    use the DFMA peak measured on this pool's B200 by tools/fp64_peak.cu."""
    mp = load_json(os.path.join(HERE, "MEASURED_PEAKS.json")) or {}
    if "fp64_tflops" in mp:
        return float(mp["fp64_tflops"]), "MEASURED_PEAKS.json"
    for name in ("r02_fp64_peak.json", "r01_fp64_peak.json"):
        pk = load_json(os.path.join(HERE, "profiles", name))
        if pk and "dfma_tflops" in pk:
            return float(pk["dfma_tflops"]), f"measured DFMA peak (profiles/{name})"
    return 37.2, "nominal 148 SM x 64 DFMA/clk x 1.965 GHz"


def hbm_peak():
    mp = load_json(os.path.join(HERE, "MEASURED_PEAKS.json")) or {}
    return next((float(v) for k, v in mp.items() if "hbm" in k.lower() and isinstance(v, (int, float))), None)


def flop_profile(workload):
    """ncu SASS FP64 counts of the pair stage of `workload` at full size
    (tools/fp64_flops.py; deterministic work)."""
    for name in (f"r02_fp64_flops_{workload}.json",):
        prof = load_json(os.path.join(HERE, "profiles", name))
        if prof and prof.get("workload") == workload:
            return prof, name
    return None, None


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle only (oracle/liboracle.so)

def oracle_context(cfg, q, seed):
    from oracle import binding as B
    P = B.OracleProblem(cfg, q, seed)
    O = B.Oracle(P.vxy, P.tri, P.p, P.coeffs, P.rules)
    return P, O, O.open()


def run_reference(args, rank, world):
    if rank != 0:
        return
    P, _O, ctx = oracle_context(args.config, args.q, args.seed)
    S = P.n_tri * len(P.rules.far[0])
    stride = args.stride or auto_stride(P.n_tgt, S)
    sub = headline_targets(P.txy, stride)
    cores = os.cpu_count() or 1
    # targets per step: about 4 s of far pairs on 16 cores (1e8 pairs/s/core)
    chunk = args.ref_chunk or int(min(len(sub), max(16, 6.4e9 / S)))
    pick = lambda k, n: sub[(np.arange(n) * max(1, len(sub) // n) + k) % len(sub)]  # noqa: E731
    for k in range(args.warmup):
        ctx.evaluate(pick(k, max(1, chunk // 8)))
    tot_t, tot_n, ms = 0.0, 0, []
    for k in range(args.steps):
        t = pick(args.warmup + k, chunk)
        t0 = time.perf_counter()
        ctx.evaluate(t)
        dt = time.perf_counter() - t0
        ms.append(1e3 * dt)
        tot_t += dt
        tot_n += len(t)
    val = tot_n / tot_t
    sample = (f"{chunk} targets per step spread over the headline subset ({len(sub)} targets: "
              f"config {args.config} in Morton order, every {stride}th), each with its full far field "
              f"({S} sources) + near + self; oracle/liboracle.so, OpenMP over targets")
    out = {
        "metric": "potential targets/sec (fp64)", "value": val, "unit": "targets/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(ms)), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (oracle's own seeded generators, SURVEY.md §8(d))",
        "impl": "reference",
        "config": workload_config(args.config, P.n_tri, P.p, P.q, P.eps, args.seed, P.n_tgt, S, stride,
                                  len(sub), world),
        "cpu_baseline": {"value": val, "unit": "targets/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "targets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# B200 arm

def ctypes_ptr(t, ptype):
    return ctypes.cast(ctypes.c_void_p(t.data_ptr()), ptype)


def timed_steps(step, n, stream, flush, dist, world):
    """n device-timed steps (CUDA events on the launching stream, L2 flushed
    between steps, barrier + synchronize on both sides, max over ranks)."""
    import torch
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    stats = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(n):
        flush.zero_()
        starts[k].record(stream)
        stats.append(step())
        ends[k].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t = torch.tensor([float(sum(ms))], dtype=torch.float64, device=flush.device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), ms, stats


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2205_04401_b200 as vp
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    pr = vp.load_config(args.config, args.q, args.seed)
    len_q = len(pr.rules.far[0])
    S = pr.n_tri * len_q
    stride = args.stride or auto_stride(pr.n_tgt, S)
    ev = vp.Evaluator(local).load(pr)
    if args.near_cache_gb or args.near_cache_depth != 3:
        ev.set_near_cache(args.near_cache_depth, int(args.near_cache_gb * (1 << 30)))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    # a non-default stream: the library orders its work (and launches the
    # captured graph) on the caller's stream, which the legacy default stream
    # would not give it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    cfg = workload_config(args.config, pr.n_tri, pr.p, pr.q, pr.eps, args.seed, pr.n_tgt, S, stride,
                          0, world)
    out = {}
    u_direct = None

    if world > 1:  # the library's own NCCL communicator carries the gather of u
        uid = [vp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ev.comm_init(world, rank, uid[0])

    def sharded(txy):
        """This rank's shard of a job: vp_shard_plan's Morton order and
        cost-balanced bounds (for the far method currently set); at N = 1 the
        job itself.  Returns (targets, bounds, order)."""
        if world == 1:
            return np.ascontiguousarray(txy), np.array([0, len(txy)]), None
        order, bounds, _ = ev.shard_plan(txy, world)
        return np.ascontiguousarray(txy[order[bounds[rank]:bounds[rank + 1]]]), bounds, order

    def device_step(d_txy, d_u, n, bounds):
        d_all = torch.empty(int(bounds[-1]) if world > 1 else 1, dtype=torch.float64, device=dev)

        def step():
            st = ev.evaluate_device(n, d_txy.data_ptr(), d_u.data_ptr(), stream.cuda_stream)
            if world > 1:  # the only collective: all-gather of u (vp_gather, NCCL)
                ev.gather(bounds, d_u.data_ptr(), d_all.data_ptr(), stream.cuda_stream)
            return st
        return step

    if args.mode == "all":
        sub = headline_targets(pr.txy, stride)
        cfg["targets"] = int(len(sub))
        ev.set_far_method("direct")
        mine, sub_bounds, _ = sharded(sub)
        T = len(mine)
        # ---- parity gate + cpu_baseline: rank 0's u against the oracle (own generators)
        cpu = check = None
        if rank == 0 and not args.no_cpu_baseline:
            pick = sub[(np.arange(CHECK_SAMPLE) * max(1, len(sub) // CHECK_SAMPLE)) % len(sub)]
            u_g, _ = ev.evaluate(pick)
            _P, _O, octx = oracle_context(args.config, args.q, args.seed)
            t0 = time.perf_counter()
            u_o, _, _ = octx.evaluate(pick)
            dt = time.perf_counter() - t0
            err = float(np.abs(u_g - u_o).max() / np.abs(u_o).max())
            check = {"targets": CHECK_SAMPLE, "max_rel_err": err, "tol": CHECK_TOL,
                     "oracle": "oracle/liboracle.so from the oracle's own generators"}
            if not err <= CHECK_TOL:
                raise SystemExit(f"bench: u differs from the oracle by {err:.3e} > {CHECK_TOL} (rel max-norm)")
            if world == 1:
                cpu = {"value": CHECK_SAMPLE / dt, "unit": "targets/s", "cores": os.cpu_count() or 1,
                       "kind": "port",
                       "sample": f"{CHECK_SAMPLE} targets spread over the headline subset, full far ({S} sources)"
                                 f" + near + self per target, oracle/liboracle.so OpenMP, {dt:.1f} s"}
            del octx
        d_txy = torch.from_numpy(mine).to(dev).contiguous()
        d_u = torch.empty(max(T, 1), dtype=torch.float64, device=dev)
        step = device_step(d_txy, d_u, T, sub_bounds)
        clk = ClockSampler(local)
        clk.start()
        clk.wait_first()
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        host_t0 = time.perf_counter()
        ms_total, ms_steps, stats = timed_steps(step, args.steps, stream, flush, dist, world)
        clk.mark(host_t0, time.perf_counter())
        clocks = clk.stop()
        value = len(sub) * args.steps / (ms_total * 1e-3)
        far_ms = float(np.mean([s["t_far_kernel_ms"] for s in stats]))
        far_flop = FAR_FLOP_PER_PAIR * T * S
        peak, peak_src = fp64_peak()
        achieved = far_flop / (far_ms * 1e-3) / 1e12
        kprof = load_json(os.path.join(HERE, "profiles", f"r02_far_kernel_{cfg['workload']}.json")) or {}
        kmatch = kprof.get("workload") == cfg["workload"] and kprof.get("targets") == T
        s0 = stats[-1]

        # ---- e2e through the public C-ABI with pinned host buffers
        n_e2e = max(1, min(args.steps, 5))
        coeffs_pin = torch.from_numpy(pr.coeffs).pin_memory()
        txy_pin = torch.from_numpy(mine).pin_memory()
        u_pin = torch.empty(max(T, 1), dtype=torch.float64).pin_memory()
        L = vp._lib.lib()
        cptr = vp._lib.c_double_p

        def e2e_step():
            rc = L.vp_set_density(ev._h, pr.p, ctypes_ptr(coeffs_pin, cptr))
            assert rc == 0, ev._err()
            st = vp._lib.VpStats()
            rc = L.vp_evaluate(ev._h, T, ctypes_ptr(txy_pin, cptr), ctypes_ptr(u_pin, cptr), ctypes.byref(st))
            assert rc == 0, ev._err()
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": len(sub) * n_e2e / float(tt.item()), "unit": "targets/s",
               "h2d_bytes_per_step": int(pr.coeffs.nbytes + mine.nbytes), "d2h_bytes_per_step": int(8 * T),
               "steps": n_e2e, "path": "vp_set_density + vp_evaluate (host buffers, C-ABI)"}
        u_direct = d_u[:T].cpu().numpy() if world == 1 else None
        del d_txy, d_u
        out.update({
            "metric": "potential targets/sec (fp64)", "value": value, "unit": "targets/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_total / args.steps, "step_ms_min": min(ms_steps), "step_ms_max": max(ms_steps),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, SURVEY.md §8(d))",
            "config": cfg,
            "split_ms": {"lib_device_total": float(np.mean([s["t_total_ms"] for s in stats])),
                         "list": float(np.mean([s["t_list_ms"] for s in stats])),
                         "sources": float(np.mean([s["t_sources_ms"] for s in stats])),
                         "far": far_ms, "pair_stage": float(np.mean([s["t_pair_ms"] for s in stats]))},
            "counts": {"targets_per_gpu": T, "near_pairs": s0["n_near_pairs"], "self_pairs": s0["n_self"],
                       "leaves": s0["n_leaves"], "panels": s0["n_panels"], "outside": s0["n_outside"]},
            "roofline": {"bound": "fp64", "kernel": "k_far (K2 direct far sum)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_source": peak_src, "flop_per_launch": far_flop, "flop_per_pair": FAR_FLOP_PER_PAIR,
                         "pairs_per_launch": T * S, "pairs_per_s": T * S / (far_ms * 1e-3),
                         "survey_flop_per_pair": SURVEY_FAR_FLOP_PER_PAIR,
                         "survey_equiv_tflops": SURVEY_FAR_FLOP_PER_PAIR * T * S / (far_ms * 1e-3) / 1e12,
                         "flop_per_pair_ncu": kprof.get("flop_per_pair_ncu") if kmatch else None,
                         "traffic": kprof.get("dram_bytes_per_launch") if kmatch else None,
                         "traffic_source": kprof.get("source") if kmatch else None},
            "gpu_launches": int(sum(s["gpu_launches"] for s in stats)),
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu, "oracle_check": check,
        })

    # ---- pair stage at full size: corrections of every target (far method none)
    full = None
    if not args.no_pairs or not args.no_fmm or args.mode == "pairs":
        full_job = headline_targets(pr.txy, 1)
    if args.mode == "pairs" or not args.no_pairs:
        ev.set_far_method("none")
        full, fb, _ = sharded(full_job)
        d_full = torch.from_numpy(full).to(dev).contiguous()
        d_uf = torch.empty(max(len(full), 1), dtype=torch.float64, device=dev)
        fstep = device_step(d_full, d_uf, len(full), fb)
        n_w = 1 if args.mode == "pairs" else 2
        for _ in range(n_w):
            fstep()
        torch.cuda.synchronize()
        n_p = args.steps if args.mode == "pairs" else max(1, min(args.steps, 10))
        p_ms, _, p_st = timed_steps(fstep, n_p, stream, flush, dist, world)
        pair_ms = float(np.mean([s["t_pair_ms"] for s in p_st]))
        s0 = p_st[-1]
        n_pairs = s0["n_near_pairs"] + s0["n_self"]
        pstage = {"targets": pr.n_tgt, "targets_per_gpu": len(full), "ms_per_step": p_ms / n_p,
                  "pair_stage_ms": pair_ms, "list_ms": float(np.mean([s["t_list_ms"] for s in p_st])),
                  "near_pairs": s0["n_near_pairs"], "self_pairs": s0["n_self"], "leaves": s0["n_leaves"],
                  "panels": s0["n_panels"], "near_pair_integrals_per_s": world * n_pairs / (pair_ms * 1e-3),
                  "what": "far method 'none': lists + near (K4) + self (K5) + point sums + assembly of all targets"}
        # list build against HBM (SURVEY.md §8(d) bytes: targets 16T, S 4T, offsets
        # 8(T+1), ids 4 P_near, element models 112 E)
        lb = 16 * len(full) + 4 * len(full) + 8 * (len(full) + 1) + 4 * s0["n_near_pairs"] + 112 * pr.n_tri
        pstage["list_build"] = {"ms": pstage["list_ms"], "bytes": lb,
                                "GBps": lb / (pstage["list_ms"] * 1e-3) / 1e9, "hbm_peak_GBps": hbm_peak()}
        prof, pname = flop_profile(cfg["workload"])
        peak, peak_src = fp64_peak()
        if prof and prof.get("targets") == len(full):
            nf = float(prof["near_stage_fp64_flops"])
            ach = nf / (pair_ms * 1e-3) / 1e12
            pstage["roofline_near"] = {
                "bound": "fp64", "kernels": ", ".join(prof["near_stage_kernels"]), "achieved": ach, "peak": peak,
                "unit": "TFLOP/s", "frac": ach / peak, "flop_per_step": nf, "stage_ms": pair_ms,
                "flop_source": f"ncu SASS dfma/dadd/dmul/DMMA counts, profiles/{pname}",
                "per_kernel_frac_ncu": {k: round(v["fp64_flops"] / (v["ncu_ms"] * 1e-3) / 1e12 / peak, 3)
                                        for k, v in prof["kernels"].items()
                                        if k in prof["near_stage_kernels"] and v["fp64_flops"] > 1e9}}
        sfl = survey_near_self_flops(s0, pr.p, len_q, len(pr.rules.near[0]), len(pr.rules.gl[0]),
                                     len(pr.rules.ggq[0]))
        if sfl:
            pstage["survey_flop_per_step"] = sfl
            pstage["survey_equiv_tflops"] = sfl / (pair_ms * 1e-3) / 1e12
        # the same evaluation replayed from its captured CUDA graph (vp_evaluate_graph:
        # no host round trip inside); replay time against the eager stage sum
        gstep = lambda: ev.evaluate_graph(len(full), d_full.data_ptr(), d_uf.data_ptr(), stream.cuda_stream)  # noqa: E731
        for _ in range(2):
            gstep()
        ev.graph_status(stream.cuda_stream)
        g_ms, _, _ = timed_steps(gstep, n_p, stream, flush, dist, world)
        ev.graph_status(stream.cuda_stream)
        pstage["graph_ms_per_step"] = g_ms / n_p
        pstage["eager_device_ms_per_step"] = float(np.mean([s["t_total_ms"] for s in p_st]))
        out["near_pair_integrals_per_s"] = pstage["near_pair_integrals_per_s"]
        out["pair_stage"] = pstage

    # ---- full evaluation of every target with the FMM far field
    if args.mode == "all" and not args.no_fmm:
        ev.set_far_method("fmm")
        full, fb, _ = sharded(full_job)
        d_full = torch.from_numpy(full).to(dev).contiguous()
        d_uf = torch.empty(max(len(full), 1), dtype=torch.float64, device=dev)
        fstep = device_step(d_full, d_uf, len(full), fb)
        for _ in range(2):
            fstep()
        torch.cuda.synchronize()
        n_f = max(1, min(args.steps, 10))
        f_ms, _, f_st = timed_steps(fstep, n_f, stream, flush, dist, world)
        out["alt_far_method"] = {
            "far_method": "fmm", "targets": pr.n_tgt, "value": pr.n_tgt * n_f / (f_ms * 1e-3),
            "ms_per_step": f_ms / n_f, "far_ms": float(np.mean([s["t_far_ms"] for s in f_st])),
            "pair_stage_ms": float(np.mean([s["t_pair_ms"] for s in f_st])),
            "fmm_levels": f_st[-1]["fmm_levels"], "fmm_order": 31,
            "gpu_launches_per_step": int(f_st[-1]["gpu_launches"])}
        if world == 1 and u_direct is not None:  # FMM vs the headline's direct u on the subset targets
            u_f = d_uf[::stride].cpu().numpy()[:len(u_direct)]
            out["alt_far_method"]["max_rel_diff_u_vs_direct_on_subset"] = float(
                np.abs(u_f - u_direct).max() / np.abs(u_direct).max())
        ev.set_far_method("direct")

    if rank == 0:
        if args.mode == "pairs":
            out = {"mode": "pairs", **out}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
