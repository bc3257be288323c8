"""ncu --set full of the headline K2 launch (GPU box):

  python tools/far_profile.py OUT.json [bench args...]

profiles the first k_far launch of `bench.py --steps 1 --warmup 3
--no-cpu-baseline --no-pairs --no-fmm` and writes the per-launch DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum), the executed FP64 flops per
pair from the SASS counters (2 per DFMA, 1 per DADD/DMUL) and the duration;
bench.py reports them as roofline.traffic / roofline.flop_per_pair_ncu when
the workload and target count match."""
import csv
import io
import json
import subprocess
import sys

EXTRA = ["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
         "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]


def main():
    out = sys.argv[1]
    cmd = [sys.executable, "bench.py", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-pairs",
           "--no-fmm"] + sys.argv[2:]
    rep = out.replace(".json", "")
    run = subprocess.run(["ncu", "--set", "full", "--metrics", ",".join(EXTRA), "--clock-control", "none",
                          "--import-source", "on", "--kernel-name-base", "function", "-k", "regex:k_far$",
                          "-c", "1", "-f", "-o", rep] + cmd, check=True, stdout=subprocess.PIPE, text=True)
    line = [l for l in run.stdout.splitlines() if l.startswith("{")][-1]
    bj = json.loads(line)
    raw = subprocess.run(["ncu", "-i", rep + ".ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units, v = r[0], r[1], r[2]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-6,
             "usecond": 1e-3, "msecond": 1.0, "second": 1e3}

    def g(k):  # value in bytes, or in ms for durations
        i = h.index(k)
        return float(v[i].replace(",", "")) * scale.get(units[i], 1.0)
    T = bj["counts"]["targets_per_gpu"]
    S = bj["config"]["sources"]
    fl = 2 * g(EXTRA[0]) + g(EXTRA[1]) + g(EXTRA[2])
    doc = {"workload": bj["config"]["workload"], "targets": T, "sources": S,
           "kernel": "k_far<false> (K2 direct far sum)",
           "source": f"ncu --set full --clock-control none, first k_far launch of {' '.join(cmd[1:])}",
           "dram_bytes_read": g("dram__bytes_read.sum"), "dram_bytes_write": g("dram__bytes_write.sum"),
           "dram_bytes_per_launch": g("dram__bytes_read.sum") + g("dram__bytes_write.sum"),
           "fp64_flops": fl, "flop_per_pair_ncu": fl / (T * S),
           "duration_ms": g("gpu__time_duration.sum"),
           "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
