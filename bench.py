#!/usr/bin/env python
"""Benchmark of the volume-potential hot path (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W --config 2 --impl b200|reference]

One step = one full evaluation pass (K1 strengths, K3 near-field lists, K2
direct far sum, K4 near pairs, K5 self pairs, assembly) over one batch of
targets: BASELINE config 2 (unit disk, 4,096 triangles, p=8, q=16, 184,320
staggered targets, seeded synthetic density) unless --config says otherwise.

Multi-GPU (torchrun, one process per GPU): weak scaling.  The job's targets
are N copies of config 2's staggered target mesh, copy r rotated by r/N of
the finest angular cell; they are Morton-ordered and cut into N contiguous
equal shards (paper_2205_04401_b200.dist), mesh and density replicated, and
the only collective is the NCCL all-gather of u (north_star).  Timing is on
the device (CUDA events) and the reported time is the max over ranks.

--impl reference times the CPU oracle (oracle/, a restatement of the
reference's specified path; the reference itself has no implementation of
it) on all host cores over a bounded target sample.
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
# 7 FMA (2 flops) + 3 add/mul (1 flop) = 17 flops.  (The exponent's
# int->double conversion runs on the XU pipe.)  The ncu SASS counters of K2
# (profiles/r01_fp64_flops_config2.json) must agree: flop_per_pair_ncu.
FAR_FLOP_PER_PAIR = 17
FP64_FLOPS_PROFILE = os.path.join(HERE, "profiles", "r01_fp64_flops_config2.json")
# SURVEY.md §8(d) frozen algorithmic work of the near and self pairs (a direct
# implementation: Koornwinder evaluation at every leaf / panel node), with
# K_p the counted cost of one Koornwinder evaluation
SURVEY_KP = {4: 117, 6: 226, 8: 371, 12: 769}


def survey_near_self_flops(st, p, len_q, len_n=49, n_l=16, n_g1=9):
    kp = SURVEY_KP.get(p)
    if kp is None:
        return None
    m2 = (p + 1) * (p + 2)
    return (st["n_leaves"] * len_n * (m2 + 60) + st["n_near_pairs"] * len_q * 51
            + st["n_panels"] * n_l * (60 + n_g1 * (kp + m2 + 10)) + st["n_self"] * len_q * 51)
# SURVEY.md §8(d)'s frozen figure counted the libdevice log (51 flops/pair);
# reported beside the roofline for comparison.
SURVEY_FAR_FLOP_PER_PAIR = 51


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--q", type=int, default=0, help="far order override (config 5 sweep)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--far", choices=["direct", "fmm"], default="direct",
                    help="far-field method of the headline measurement (north_star: direct)")
    ap.add_argument("--no-fmm", action="store_true", help="skip the secondary FMM measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-stride", type=int, default=8, help="cpu_baseline target sample stride")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def rotate(txy, theta):
    c, s = np.cos(theta), np.sin(theta)
    return np.stack([c * txy[:, 0] - s * txy[:, 1], s * txy[:, 0] + c * txy[:, 1]], 1)


def job_targets(pr, world):
    """The whole job's targets for weak scaling: world copies of the config's
    target set, copy r rotated by r/world of the finest angular cell (disk
    configs) or shifted by r/world of a cell width, so every GPU gets a
    config-sized batch of distinct targets."""
    if world == 1:
        return pr.txy.copy()
    parts = []
    for r in range(world):
        if r == 0:
            parts.append(pr.txy)
        elif pr.config == 2:
            parts.append(rotate(pr.txy, 2 * np.pi / (16 * 16) * r / world))
        else:
            h = np.sqrt(2.0 / pr.n_tri)
            parts.append(pr.txy + np.array([h * r / world * 0.37, h * r / world * 0.21]))
    return np.concatenate(parts)


def rank_targets(pr, rank, world):
    """This rank's shard (north_star): the job's targets in
    Morton order, cut into contiguous equal-count shards
    (paper_2205_04401_b200.dist); mesh and density are replicated."""
    from paper_2205_04401_b200.dist import morton_order, shard_bounds
    U = job_targets(pr, world)
    if world == 1:
        return U, len(U)
    order = morton_order(U)
    lo, hi = shard_bounds(len(U), rank, world)
    return U[order[lo:hi]], len(U)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []  # (host time, fields)
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
        """nvidia-smi's start-up (NVML init) can stall CUDA calls of this
        process, so it is started before the warm-up and the timed region
        begins only after its first sample."""
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
        if self.window is not None:  # samples taken during the timed region (+ one period)
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
    pk = load_json(os.path.join(HERE, "profiles", "r01_fp64_peak.json"))
    if pk and "dfma_tflops" in pk:
        return float(pk["dfma_tflops"]), "measured DFMA peak (profiles/r01_fp64_peak.json)"
    return 37.2, "nominal 148 SM x 64 DFMA/clk x 1.965 GHz"


def cpu_baseline(pr, stride, threads=0):
    from oracle.binding import Oracle
    O = Oracle.from_problem(pr)
    sub = pr.txy[::stride]
    t0 = time.perf_counter()
    O.evaluate(sub, nthreads=threads)
    dt = time.perf_counter() - t0
    return len(sub), dt


def run_reference(args, pr, rank, world):
    """--impl reference: the CPU oracle on all host cores, bounded samples."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    stride = max(1, pr.n_tgt // 2880)  # ~2.9k targets per step (~1 s on 16 cores)
    for _ in range(args.warmup):
        cpu_baseline(pr, stride * 4)
    tot_t, tot_n = 0.0, 0
    for _ in range(args.steps):
        n, dt = cpu_baseline(pr, stride)
        tot_t += dt
        tot_n += n
    val = tot_n / tot_t
    sample = f"every {stride}th target of config {pr.config} ({pr.n_tgt // stride} of {pr.n_tgt}) per step, full far+near+self"
    out = {
        "metric": "potential targets/sec (fp64)", "value": val, "unit": "targets/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, SURVEY.md §8(d))",
        "impl": "reference",
        "config": {"workload": f"config{pr.config}", "n_tri": pr.n_tri, "p": pr.p, "q": pr.q,
                   "eps": pr.eps, "targets_per_step": pr.n_tgt // stride},
        "cpu_baseline": {"value": val, "unit": "targets/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": val, "unit": "targets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    import paper_2205_04401_b200 as vp
    from paper_2205_04401_b200.dist import gather_potentials
    pr = vp.load_config(args.config, args.q, args.seed)
    if args.impl == "reference":
        run_reference(args, pr, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    ev = vp.Evaluator(local).load(pr)
    ev.set_far_method(args.far)
    txy_h, T_job = rank_targets(pr, rank, world)
    T = txy_h.shape[0]
    d_txy = torch.from_numpy(txy_h).to(dev).contiguous()
    d_u = torch.empty(T, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    def step():
        st = ev.evaluate_device(T, d_txy.data_ptr(), d_u.data_ptr(), stream.cuda_stream)
        if world > 1:  # the only collective: gather of u (NCCL all-gather of padded shards)
            gather_potentials(d_u, T_job, rank, world)
        return st

    clk = ClockSampler(local)
    clk.start()
    clk.wait_first()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # ---- timed region: K device-timed steps, L2 flushed between steps ----
    host_t0 = time.perf_counter()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stats = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        starts[k].record(stream)
        stats.append(step())
        ends[k].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk.mark(host_t0, time.perf_counter())
    clocks = clk.stop()
    ms_steps = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_total = float(sum(ms_steps))
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_per_step = ms_total / args.steps
    value = T_job * args.steps / (ms_total * 1e-3)  # the whole job's targets

    # far kernel (dominant) roofline from the library's device events
    S = stats[-1]["n_sources"]
    far_ms = float(np.mean([s["t_far_kernel_ms"] for s in stats]))
    far_flop = FAR_FLOP_PER_PAIR * T * S
    peak, peak_src = fp64_peak()
    achieved = far_flop / (far_ms * 1e-3) / 1e12
    prof = load_json(os.path.join(HERE, "profiles", "far_kernel_traffic.json")) or {}
    # pair stage: near chain (main stream) beside self + point sums (s3)
    pair_ms = float(np.mean([s["t_pair_ms"] for s in stats]))
    n_pairs = stats[-1]["n_near_pairs"] + stats[-1]["n_self"]

    # e2e through the public API with pinned host buffers (set_density + evaluate)
    e2e = None
    if rank == 0 or world > 1:
        coeffs_pin = torch.from_numpy(pr.coeffs).pin_memory()
        txy_pin = torch.from_numpy(txy_h).pin_memory()
        u_pin = torch.empty(T, dtype=torch.float64).pin_memory()
        L = vp._lib.lib()
        cptr = vp._lib.c_double_p

        def e2e_step():
            rc = L.vp_set_density(ev._h, pr.p, ctypes_ptr(coeffs_pin, cptr))
            assert rc == 0, ev._err()
            st = vp._lib.VpStats()
            rc = L.vp_evaluate(ev._h, T, ctypes_ptr(txy_pin, cptr), ctypes_ptr(u_pin, cptr),
                               ctypes.byref(st))
            assert rc == 0, ev._err()
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        e2e = {"value": T_job * args.steps / dt, "unit": "targets/s",
               "h2d_bytes_per_step": int(pr.coeffs.nbytes + txy_h.nbytes),
               "d2h_bytes_per_step": int(8 * T)}

    # secondary: the same steps with the other far-field method (FMM)
    alt = None
    if not args.no_fmm:
        other = "fmm" if args.far == "direct" else "direct"
        u_ref = d_u.clone()
        ev.set_far_method(other)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a_st, a_ms = [], []
        for k in range(args.steps):
            flush.zero_()
            starts[k].record(stream)
            a_st.append(step())
            ends[k].record(stream)
        torch.cuda.synchronize()
        a_ms = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
        ta = torch.tensor([a_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ta, op=dist.ReduceOp.MAX)
        a_ms = float(ta.item())
        diff = float((d_u - u_ref).abs().max().item() / u_ref.abs().max().item())
        alt = {"far_method": other, "value": T_job * args.steps / (a_ms * 1e-3),
               "ms_per_step": a_ms / args.steps,
               "far_ms": float(np.mean([s["t_far_ms"] for s in a_st])),
               "fmm_levels": a_st[-1]["fmm_levels"], "fmm_order": 31,
               "max_rel_diff_u_vs_headline": diff}
        ev.set_far_method(args.far)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n, dt = cpu_baseline(pr, args.cpu_stride)
        cpu = {"value": n / dt, "unit": "targets/s", "cores": os.cpu_count() or 1, "kind": "port",
               "sample": f"every {args.cpu_stride}th target of config {pr.config} ({n} of {pr.n_tgt}), "
                         f"full far+near+self per target, oracle/liboracle.so OpenMP, {dt:.1f} s"}

    # near field (K4 + K5 stages): executed FP64 flops per step from the ncu
    # SASS counters of the same configuration (deterministic work), over the
    # live device time of those stages
    roof_near = None
    prof_fl = load_json(FP64_FLOPS_PROFILE)
    if prof_fl and pr.config == 2 and not args.q and args.seed == 0 and not prof_fl.get("config_args"):
        nf = float(prof_fl["near_stage_fp64_flops"])
        ach = nf / (pair_ms * 1e-3) / 1e12
        kf = prof_fl["kernels"].get("k_far<0>") or prof_fl["kernels"].get("k_far<false>")
        roof_near = {"bound": "fp64", "kernels": "near + self stages (" + ", ".join(prof_fl["near_stage_kernels"]) + ")",
                     "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                     "flop_per_step": nf, "stage_ms": pair_ms,
                     "flop_source": "ncu SASS dfma/dadd/dmul/DMMA counts, profiles/r01_fp64_flops_config2.json",
                     "per_kernel_frac_ncu": {k: round(v["fp64_flops"] / (v["ncu_ms"] * 1e-3) / 1e12 / peak, 3)
                                             for k, v in prof_fl["kernels"].items()
                                             if k in prof_fl["near_stage_kernels"] and v["fp64_flops"] > 1e9}}
    else:
        kf = None
    sfl = survey_near_self_flops(stats[-1], pr.p, pr_len_q(pr), len(pr.rules.near[0]), len(pr.rules.gl[0]),
                                 len(pr.rules.ggq[0]))
    if roof_near is not None and sfl is not None:
        roof_near["survey_flop_per_step"] = sfl
        roof_near["survey_equiv_tflops"] = sfl / (pair_ms * 1e-3) / 1e12

    if rank == 0:
        s0 = stats[-1]
        list_ms = float(np.mean([s["t_list_ms"] for s in stats]))
        list_bytes = 16 * T + 4 * T + 8 * (T + 1) + 4 * s0["n_near_pairs"] + 112 * pr.n_tri
        try:
            with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
                mp = json.load(f)
            hbm_peak = next((float(v) for k, v in mp.items() if "hbm" in k.lower() and isinstance(v, (int, float))),
                            None)
        except (OSError, ValueError):
            hbm_peak = None
        out = {
            "metric": "potential targets/sec (fp64)", "value": value, "unit": "targets/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_per_step, "step_ms_min": min(ms_steps), "step_ms_max": max(ms_steps),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, SURVEY.md §8(d)); L2 flushed between timed steps",
            "config": {"workload": f"config{pr.config}", "n_tri": pr.n_tri, "p": pr.p, "q": pr.q,
                       "eps": pr.eps, "targets_per_gpu": T, "sources": S, "seed": args.seed,
                       "near_pairs": s0["n_near_pairs"], "self_pairs": s0["n_self"],
                       "l2": "flushed (256 MB write) between timed steps",
                       "parallelism": f"weak x{world} (targets sharded, mesh+density replicated)"},
            "near_pair_integrals_per_s": world * n_pairs / (pair_ms * 1e-3),
            # K3 list build against HBM (SURVEY.md §8(d) bytes: targets 16T, S 4T, offsets
            # 8(T+1), ids 4 P_near, element models 112 E); at config 2 it is launch/latency
            # bound (two tiny passes + a scan), so this is reported, not a roofline claim
            "list_build": {"ms": list_ms, "bytes": list_bytes,
                           "GBps": list_bytes / (list_ms * 1e-3) / 1e9,
                           "hbm_peak_GBps": hbm_peak},
            "split_ms": {"lib_device_total": float(np.mean([s["t_total_ms"] for s in stats])),
                         "list": float(np.mean([s["t_list_ms"] for s in stats])),
                         "sources": float(np.mean([s["t_sources_ms"] for s in stats])),
                         "far": far_ms,
                         "near": float(np.mean([s["t_near_ms"] for s in stats])),
                         "self": float(np.mean([s["t_self_ms"] for s in stats])),
                         "pair_stage": pair_ms},
            # slowest step's stages (host round trips inside a stage show up here)
            "split_ms_max": {k: float(max(s[f"t_{k}_ms"] for s in stats)) for k in ("list", "far", "near", "self", "pair")},
            "roofline": {"bound": "fp64", "kernel": "k_far (K2 direct far sum)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "flop_per_launch": far_flop, "flop_per_pair": FAR_FLOP_PER_PAIR,
                         "pairs_per_s": T * S / (far_ms * 1e-3),
                         "survey_flop_per_pair": SURVEY_FAR_FLOP_PER_PAIR,
                         "survey_equiv_tflops": SURVEY_FAR_FLOP_PER_PAIR * T * S / (far_ms * 1e-3) / 1e12,
                         "flop_per_pair_ncu": (kf["fp64_flops"] / (T * S)) if kf else None,
                         "traffic": prof.get("dram_bytes_per_launch"),
                         "traffic_source": prof.get("source")},
            "roofline_near": roof_near,
            "far_method": args.far,
            "alt_far_method": alt,
            "gpu_launches": int(sum(s["gpu_launches"] for s in stats)),
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pr_len_q(pr):
    """far-rule length of a problem (the sources per element)"""
    return int(len(pr.rules.far[0]))


def ctypes_ptr(t, ptype):
    return ctypes.cast(ctypes.c_void_p(t.data_ptr()), ptype)


if __name__ == "__main__":
    main()
