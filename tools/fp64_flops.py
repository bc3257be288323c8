"""Executed FP64 work of every kernel of one evaluation step, from ncu SASS
counters (run on the GPU box):

  python tools/fp64_flops.py OUT.json [bench args...]

runs `ncu --metrics <duration, dfma/dadd/dmul thread counts>` over
`bench.py --mode pairs --steps 1 --warmup 1` (the full-size pair stage:
far method none) and writes, per
kernel, the FP64 flops of one launch (2 per DFMA, 1 per DADD/DMUL, the
tensor-pipe FP64 ops of DMMA; medians
over the run's launches -- every step does identical work) and its ncu
duration.  bench.py turns the near-stage totals into the near-field
roofline with its own live timing (the ncu durations are cold-cache and
serialised, kept for the per-kernel share only)."""
import csv
import io
import json
import os
import statistics
import subprocess
import sys

MET = {"gpu__time_duration.sum": "ns",
       "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
       "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
       "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
       "sm__ops_path_tensor_src_fp64.sum": "dmma"}  # DMMA flops (2 per FMA)
# kernels of the near field (K4) and self (K5) stages of an evaluation
NEAR_STAGE = ("k_near_leaves", "k_leaves_copy", "k_near_cache", "k_near_cache_mma", "k_near_cache_mma2", "k_near_c8", "k_near_cg", "k_near_ct", "k_near_int",
              "k_psum_tgt", "k_self", "k_near_combine", "k_pair_tgt")


def main():
    out = sys.argv[1]
    cmd = [sys.executable, "bench.py", "--mode", "pairs", "--steps", "1", "--warmup", "1"] + sys.argv[2:]
    log = "/tmp/fp64_flops.csv"
    run = subprocess.run(["ncu", "--metrics", ",".join(MET), "--clock-control", "none", "--csv",
                          "--log-file", log] + cmd, check=True, stdout=subprocess.PIPE, text=True)
    line = [l for l in run.stdout.splitlines() if l.startswith("{")][-1]
    bj = json.loads(line)["pair_stage"]
    rows = list(csv.reader(io.StringIO(open(log).read())))
    h = None
    per = {}
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            h = {n: i for i, n in enumerate(r)}
            continue
        if h is None or len(r) < len(h):
            continue
        name = r[h["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        met = r[h["Metric Name"]]
        if met not in MET:
            continue
        val = float(r[h["Metric Value"]].replace(",", ""))
        lid = r[h["ID"]]
        per.setdefault(name, {}).setdefault(lid, {})[MET[met]] = val
    res = {}
    for name, launches in per.items():
        fl = [2 * v.get("dfma", 0) + v.get("dadd", 0) + v.get("dmul", 0) + v.get("dmma", 0) for v in launches.values()]
        ns = [v.get("ns", 0) for v in launches.values()]
        res[name] = {"launches": len(fl), "fp64_flops": statistics.median(fl), "ncu_ms": statistics.median(ns) * 1e-6}
    near = {k: v for k, v in res.items() if k.split("<")[0] in NEAR_STAGE}
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "4"
    doc = {"how": "ncu --metrics " + ",".join(MET) + " over " + " ".join(cmd[1:]),
           "config_args": sys.argv[2:], "workload": f"config{cfg}", "targets": bj["targets_per_gpu"],
           "kernels": res,
           "near_stage_fp64_flops": sum(v["fp64_flops"] for v in near.values()),
           "near_stage_kernels": sorted(near)}
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    json.dump(doc, open(out, "w"), indent=1)
    for k, v in sorted(res.items(), key=lambda kv: -kv[1]["fp64_flops"]):
        if v["fp64_flops"]:
            print(f"{k:40s} {v['fp64_flops']:.4e} flop  {v['ncu_ms']:8.3f} ms  "
                  f"{v['fp64_flops'] / (v['ncu_ms'] * 1e-3) / 1e12:6.2f} TFLOP/s")


if __name__ == "__main__":
    main()
