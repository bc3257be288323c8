#!/bin/bash
# FP64 peak on the box with the SM clock sampled during the run (GPU box).
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu
nvidia-smi -i 0 --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > gpurun_out/fp64_peak_smi.csv &
SMI=$!
/tmp/fp64_peak > gpurun_out/fp64_peak.json
kill $SMI
python - <<'PY'
import json, statistics
d = json.load(open("gpurun_out/fp64_peak.json"))
rows = [l.split(",") for l in open("gpurun_out/fp64_peak_smi.csv") if l.strip()]
sm = [float(r[0]) for r in rows if float(r[2]) > 300]   # samples under load
d["sm_mhz_under_load_median"] = statistics.median(sm) if sm else None
d["sm_max_mhz"] = max(float(r[1]) for r in rows)
d["power_w_max"] = max(float(r[2]) for r in rows)
d["reasons_seen"] = sorted({r[3].strip() for r in rows})
d["nominal_dfma_tflops_at_max_clock"] = 148 * 64 * 2 * d["sm_max_mhz"] * 1e6 / 1e12
json.dump(d, open("gpurun_out/fp64_peak.json", "w"))
print(json.dumps(d))
PY
