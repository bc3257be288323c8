#!/bin/bash
# usage (on the GPU box): tools/prof_pairs.sh <tag> [kernel-function-name ...]
# Full-size pair stage of config 4 (bench.py --mode pairs): plain run, launch
# list, FP64 flop counts (tools/fp64_flops.py), one ncu --set full capture per
# named kernel.  Outputs in gpurun_out/.
TAG=$1; shift
CMD="python bench.py --mode pairs --steps 1 --warmup 1"
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
python tools/fp64_flops.py gpurun_out/${TAG}_fp64_flops_config4.json > gpurun_out/${TAG}_fp64_flops.log 2>&1
for K in "$@"; do
  ncu --set full --clock-control none --import-source on --kernel-name-base function -k $K -s 1 -c 1 \
      -o gpurun_out/${TAG}_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1 || true
done
