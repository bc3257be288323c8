#!/bin/bash
# usage (on the GPU box): tools/prof.sh <tag> [kernel-function-name ...]
# 1) plain run of the bench command, 2) launch list with per-kernel times,
# 3) one `ncu --set full` capture per named kernel.  Outputs in gpurun_out/.
set -e
TAG=$1; shift
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
for K in "$@"; do
  ncu --set full --clock-control none --import-source on --kernel-name-base function -k $K -s 1 -c 1 \
      -o gpurun_out/${TAG}_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1 || true
done
